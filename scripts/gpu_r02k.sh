# round 2 final sweep, part 1: GPU suite, smoke, RMAT-22/24 + power-law configs (parity, e2e, cpu_baseline)
mkdir -p gpurun_out
T=${1:-r02k}
( nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; lscpu | grep -i "model name" ) > gpurun_out/${T}_host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log | cut -c1-200
run() { n=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err; echo $n rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_$n.json | cut -c1-300; }
run cl4
run ref --impl reference --steps 2 --warmup 1
run tc --workload tc
run cl5 --workload cl5 --steps 3 --warmup 3
run c4 --workload c4 --steps 3 --warmup 3
run diamond --workload diamond --steps 3 --warmup 3
run mc3 --workload mc3
run mc4 --workload mc4 --steps 3 --warmup 3
