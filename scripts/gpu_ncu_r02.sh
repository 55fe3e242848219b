# ncu evidence per config: launch list of one step (device time per launch) and one
# `--set full` capture of the step's mining kernels. Usage: gpu_ncu_r02.sh TAG "w1 w2 ..."
mkdir -p gpurun_out
T=${1:-r02n}
WL=${2:-"cl4 tc cl5 c4 diamond mc3 mc4"}
B="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline --no-parity"
for w in $WL; do
  case $w in
    cl4|tc|cl5) RX="k_clique_" ;;
    c4*) RX="k_c4_(warp|cta|stage|stage2|grid)" ;;
    diamond) RX="k_clique_|k_sum_choose2" ;;
    tc27) RX="k_clique_" ;;
    *) RX="g2m_plan" ;;
  esac
  case $w in
    tc27) A="--workload tc --scale 27" ;;
    c425) A="--workload c4 --scale 25" ;;
    *) A="--workload $w" ;;
  esac
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_${w}_launches.csv \
    python bench.py $A $B > /dev/null 2> gpurun_out/${T}_${w}_launches.err; echo $w launches rc=$?
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c 12 \
    -o gpurun_out/${T}_${w}_full -f python bench.py $A $B > /dev/null 2> gpurun_out/${T}_${w}_full.err; echo $w full rc=$?
done
ls -la gpurun_out/ | grep ${T}
