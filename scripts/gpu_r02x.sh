mkdir -p gpurun_out
T=${1:-r02x}
for w in tc cl4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-parity > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo $w rc=$?; grep "e2e steps" gpurun_out/${T}_bench_$w.err
done
