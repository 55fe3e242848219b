# full ncu capture of the mining kernels of one bench step:
#   bash scripts/gpu_ncu_full.sh <workload> <tag> [kernel-regex] [count] [skip]
W=${1:-cl4}; TAG=${2:-rXX}; KR=${3:-"k_clique_(warp|cta)|g2m_plan"}; NC=${4:-8}; SK=${5:-0}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KR" --launch-skip $SK -c $NC \
  -o gpurun_out/${TAG}_${W}_full -f \
  python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline > gpurun_out/${TAG}_${W}_full_bench.log 2>&1
echo rc=$?; tail -3 gpurun_out/${TAG}_${W}_full_bench.log
