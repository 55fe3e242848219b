mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py -q -x -k "diamond_support or diamond_allreduce or rank_copy or orientation_tiles" > gpurun_out/z_new_tests.log 2>&1; tail -5 gpurun_out/z_new_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
G2M_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --workload diamond --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench_diamond_n2gloo.json 2> gpurun_out/z_bench_diamond_n2gloo.err; echo n2 rc=$?; python scripts/line_summary.py gpurun_out/z_bench_diamond_n2gloo.json | cut -c1-300
