mkdir -p gpurun_out
T=${1:-r02y}
timeout 900 python -m pytest tests -m gpu -q -x -k "hub_core or clique or kernel_work or lgs" > gpurun_out/${T}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_pytest.log
for w in tc cl4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-parity > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo $w rc=$?; grep "e2e steps" gpurun_out/${T}_bench_$w.err
done
