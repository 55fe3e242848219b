mkdir -p gpurun_out
timeout 900 python bench.py --workload tc --scale 27 --steps 3 --warmup 3 > gpurun_out/r02h_bench_tc27.json 2> gpurun_out/r02h_bench_tc27.err; echo tc27 rc=$?; python scripts/line_summary.py gpurun_out/r02h_bench_tc27.json | cut -c1-300
