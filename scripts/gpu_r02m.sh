# round 2: focused ncu captures with source hotspots (summarised on the box):
# cl4 after the hub core, cl5's W=16 tier, the 4-cycle staging tier on RMAT-22 with a small slab
mkdir -p gpurun_out /tmp/ncu
T=${1:-r02m}
B="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline --no-parity"
cap() {  # tag env regex skip count bench-args
  tag=$1; ENVV=$2; RX=$3; SKIP=$4; CNT=$5; shift 5
  env $ENVV timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c $CNT \
    -o /tmp/ncu/${T}_${tag} -f python bench.py "$@" $B > /dev/null 2> /tmp/ncu/${tag}.err; echo $tag full rc=$?
  ncu -i /tmp/ncu/${T}_${tag}.ncu-rep --page raw --csv 2>/dev/null | gzip -c > gpurun_out/${T}_${tag}_raw.csv.gz
  for sk in 0 1 2 3 4; do
    timeout 300 python scripts/ncu_hotspots.py /tmp/ncu/${T}_${tag}.ncu-rep "$RX" 30 $sk gpurun_out/${T}_${tag}_src${sk}.csv.gz >> gpurun_out/${T}_${tag}_hotspots.txt 2>&1
  done
  ls -la gpurun_out/${T}_${tag}*
}
case "${2:-default}" in
  default)
    cap cl4 "X=0" "k_clique_(cta|pairs)" 0 5 --workload cl4
    cap cl5w16 "X=0" "k_clique_cta" 1 1 --workload cl5
    cap c4s22 "G2M_C4_STAGE_CAP=1048576" "k_c4_stage" 0 2 --workload c4 --scale 22 ;;
  t)
    cap c4s24 "G2M_C4_STAGE_CAP=1048576" "k_c4_stage2" 0 1 --workload c4 --scale 24
    cap mc4 "X=0" "g2m_plan" 0 3 --workload mc4
    cap cl4b "X=0" "k_clique_cta" 1 1 --workload cl4 ;;
esac
du -sh gpurun_out
