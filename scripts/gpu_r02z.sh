mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "medium_density" > gpurun_out/z_gr_test.log 2>&1; tail -15 gpurun_out/z_gr_test.log
