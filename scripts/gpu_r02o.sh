# round 2: full GPU suite (FSM, LGS codegen, hub core, kernel work), then C5 4-cycle RMAT-27 with RED + 16M cap
mkdir -p gpurun_out
T=${1:-r02o}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/${T}_pytest_gpu.log
timeout 1500 python bench.py --workload c4 --scale 27 --steps 2 --warmup 3 --balg-sample 1e-5 --cpu-seconds 20 > gpurun_out/${T}_bench_c427.json 2> gpurun_out/${T}_bench_c427.err; echo c427 rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_c427.json | cut -c1-300
