# full ncu capture of selected kernels of one bench step, extra bench args after --:
#   bash scripts/gpu_ncu_args.sh <tag> <kernel-regex> <count> <skip> -- <bench args...>
TAG=$1; KR=$2; NC=$3; SK=$4; shift 5
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KR" --launch-skip $SK -c $NC \
  -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline "$@" > gpurun_out/${TAG}_full_bench.log 2>&1
echo rc=$?
