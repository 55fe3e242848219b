mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r02g_bench_cl4.json 2> gpurun_out/r02g_bench_cl4.err; echo bench rc=$?; python scripts/line_summary.py gpurun_out/r02g_bench_cl4.json | cut -c1-300
timeout 900 python bench.py --workload tc > gpurun_out/r02g_bench_tc.json 2> gpurun_out/r02g_bench_tc.err; echo tc rc=$?; python scripts/line_summary.py gpurun_out/r02g_bench_tc.json | cut -c1-300
