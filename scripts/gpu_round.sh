# full check: GPU test suite, smoke, default bench (all keys), reference arm, other configs, ncu evidence
mkdir -p gpurun_out
T=${1:-r01}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_cl4.json 2> gpurun_out/${T}_bench_cl4.err; echo bench rc=$?; cut -c1-300 gpurun_out/${T}_bench_cl4.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo ref rc=$?; cut -c1-300 gpurun_out/${T}_bench_ref.json
for w in tc cl5 c4 diamond mc3 mc4; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo $w rc=$?; cut -c1-200 gpurun_out/${T}_bench_$w.json
done
# ncu: launch list of one cold cl4 step + full capture of its mining kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_cl4_launches.csv \
  python bench.py --workload cl4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline > /dev/null 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_clique_(warp|cta|pairs)" -c 10 \
  -o gpurun_out/${T}_cl4_full -f python bench.py --workload cl4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-roofline > /dev/null 2>&1; echo full rc=$?
# config C5 on one GPU (device-generated R-MAT)
timeout 1500 python bench.py --workload tc --scale 27 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_tc27.json 2> gpurun_out/${T}_bench_tc27.err; echo tc27 rc=$?
timeout 1500 python bench.py --workload c4 --scale 25 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_c425.json 2> gpurun_out/${T}_bench_c425.err; echo c425 rc=$?
