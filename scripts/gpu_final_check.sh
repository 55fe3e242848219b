# round-end check of HEAD: full GPU suite, smoke, default bench (all keys), reference arm
mkdir -p gpurun_out
T=${1:-r01p}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_cl4.json 2> gpurun_out/${T}_bench_cl4.err; echo bench rc=$?; cut -c1-400 gpurun_out/${T}_bench_cl4.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo ref rc=$?; cut -c1-300 gpurun_out/${T}_bench_ref.json
