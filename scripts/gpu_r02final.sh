# round 2 final check of HEAD: smoke, default bench (cl4), reference arm, TC, diamond
mkdir -p gpurun_out
T=${1:-r02f}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log | cut -c1-200
run() { n=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err; echo $n rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_$n.json | cut -c1-300; }
run cl4
run ref --impl reference --steps 2 --warmup 1
run tc --workload tc
run diamond --workload diamond --steps 3 --warmup 3
