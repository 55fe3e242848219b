# round 2 sweep: full GPU suite, smoke, every config with parity/roofline/e2e/cpu_baseline, reference arm, C5
mkdir -p gpurun_out
T=${1:-r02c}
( nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; free -g; lscpu | grep -i "model name\|socket\|core" ) > gpurun_out/${T}_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log | cut -c1-200
run() { n=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err; echo $n rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_$n.json; }
run cl4
run ref --impl reference --steps 2 --warmup 1
run tc --workload tc
run cl5 --workload cl5 --steps 3 --warmup 3
run c4 --workload c4 --steps 3 --warmup 3
run diamond --workload diamond --steps 3 --warmup 3
run mc3 --workload mc3
run mc4 --workload mc4 --steps 3 --warmup 3
run tc27 --workload tc --scale 27 --steps 3 --warmup 3
run c425 --workload c4 --scale 25 --steps 2 --warmup 3
