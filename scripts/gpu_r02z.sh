mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x -k "rank or orient" > gpurun_out/z_new_tests.log 2>&1; tail -2 gpurun_out/z_new_tests.log
python scripts/e2e_debug.py cl4 > gpurun_out/z_e2e_cl4_v6.txt 2>&1; grep -h "plain\|orient\|rank build" gpurun_out/z_e2e_cl4_v6.txt | tail -10
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank|k_orient" -c 12 --csv --log-file gpurun_out/z_ncu_rank6.csv python scripts/e2e_debug.py cl4 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
