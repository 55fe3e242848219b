# ncu evidence for one bench workload: launch list (cold, serialised) + full capture of the clique kernels.
# usage: bash scripts/gpu_profile.sh <workload> <tag>
set -x
W=${1:-cl4}; TAG=${2:-r01}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_${W}_launches.csv \
  python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline > gpurun_out/${TAG}_${W}_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_clique_(warp|cta)|g2m_plan}" -c ${NCAP:-6} \
  -o gpurun_out/${TAG}_${W}_full -f \
  python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline > gpurun_out/${TAG}_${W}_full_bench.log 2>&1
ls -la gpurun_out
