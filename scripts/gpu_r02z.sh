mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x -k "rank or orient" > gpurun_out/z_new_tests.log 2>&1; tail -2 gpurun_out/z_new_tests.log
for v in 1 0; do for wl in cl4 tc; do G2M_UPLOAD_PIPE=$v python scripts/e2e_breakdown.py $wl > gpurun_out/z_pipe_${wl}_$v.txt 2>&1; echo "== pipe=$v $wl"; tail -2 gpurun_out/z_pipe_${wl}_$v.txt; done; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
