# round 2, first GPU pass: full GPU suite, smoke, default bench (parity + roofline), split simulation
mkdir -p gpurun_out
T=${1:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_cl4.json 2> gpurun_out/${T}_bench_cl4.err; echo bench rc=$?; cut -c1-400 gpurun_out/${T}_bench_cl4.json; tail -3 gpurun_out/${T}_bench_cl4.err
timeout 900 python bench.py --steps 2 --warmup 1 --simulate-parts 8 --no-cpu-baseline --no-e2e --no-parity --no-roofline > gpurun_out/${T}_sim_cl4.json 2> gpurun_out/${T}_sim_cl4.err; echo sim rc=$?; grep simulated gpurun_out/${T}_sim_cl4.err
