# round 2: full GPU suite (new LGS codegen / hub partition / least-first / staged pair / GCSR tests),
# then config C5's 4-cycle on device-generated RMAT-27 and an ncu capture of TC on RMAT-27
mkdir -p gpurun_out
T=${1:-r02e}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/${T}_pytest_gpu.log
timeout 2400 python bench.py --workload c4 --scale 27 --steps 2 --warmup 3 --balg-sample 1e-5 --cpu-seconds 20 > gpurun_out/${T}_bench_c427.json 2> gpurun_out/${T}_bench_c427.err; echo c427 rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_c427.json; tail -3 gpurun_out/${T}_bench_c427.err
