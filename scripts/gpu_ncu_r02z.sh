# ncu evidence per config, summarised ON THE BOX (reps are too large to bring back):
# launch list of one step + `--set full` capture of the step's mining kernels ->
# gpurun_out/${T}_${w}_ncu.md, gpurun_out/${T}_ncu_summary.json, hotspot text.
# Usage: gpu_ncu_r02.sh TAG "w1 w2 ..."   (w may carry env as w:VAR=VAL)
mkdir -p gpurun_out /tmp/ncu
T=${1:-r02n}
WL=${2:-"cl4 tc cl5 c4 diamond mc3 mc4"}
B="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline --no-parity"
for spec in $WL; do
  w=${spec%%:*}; ENVV=""; [ "$spec" != "$w" ] && ENVV=${spec#*:}
  tag=$w; [ -n "$ENVV" ] && tag="${w}_$(echo $ENVV | tr '=;,' '___')"
  case $w in
    cl4|tc|cl5|tc27) RX="k_clique_" ;;
    c4*) RX="k_c4_(warp|cta|stage|stage2|grid)" ;;
    diamond) RX="k_clique_|k_sum_choose2" ;;
    *) RX="g2m_plan" ;;
  esac
  case $w in
    tc27) A="--workload tc --scale 27"; KEY=tc@rmat27 ;;
    c425) A="--workload c4 --scale 25"; KEY=c4@rmat25 ;;
    c4|diamond) A="--workload $w"; KEY=$w@rmat24 ;;
    mc3|mc4) A="--workload $w"; KEY=$w@powerlaw200000 ;;
    *) A="--workload $w"; KEY=$w@rmat22 ;;
  esac
  [ -n "$ENVV" ] && KEY="$KEY[$ENVV]"
  env $ENVV timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_${tag}_launches.csv \
    python bench.py $A $B > /dev/null 2> /tmp/ncu/${tag}_launches.err; echo $tag launches rc=$?
  env $ENVV timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c 12 \
    -o /tmp/ncu/${T}_${tag}_full -f python bench.py $A $B > /dev/null 2> /tmp/ncu/${tag}_full.err; echo $tag full rc=$?
  python scripts/profile_summary.py /tmp/ncu/${T}_${tag}_full.ncu-rep "$KEY" gpurun_out/${T}_${tag}_ncu.md gpurun_out/${T}_ncu_summary.json > /dev/null 2>&1; echo $tag summary rc=$?
  :
  for sk in 0 1 2 3 4 5; do
    python scripts/ncu_hotspots.py /tmp/ncu/${T}_${tag}_full.ncu-rep "$RX" 25 $sk >> gpurun_out/${T}_${tag}_hotspots.txt 2>&1
  done
done
du -sh gpurun_out
