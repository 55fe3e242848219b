# config C5 (single GPU): TC on device-generated RMAT-27, 4-cycle on RMAT-25
mkdir -p gpurun_out
T=${1:-r01}
G2M_DEBUG=1 timeout 1500 python bench.py --workload tc --scale 27 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_tc27.json 2> gpurun_out/${T}_bench_tc27.err; echo tc27 rc=$?; cut -c1-300 gpurun_out/${T}_bench_tc27.json
G2M_DEBUG=1 timeout 1500 python bench.py --workload c4 --scale 25 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_c425.json 2> gpurun_out/${T}_bench_c425.err; echo c425 rc=$?; cut -c1-300 gpurun_out/${T}_bench_c425.json
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
