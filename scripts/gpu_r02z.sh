mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x -k "rank or orient" > gpurun_out/z_new_tests.log 2>&1; tail -2 gpurun_out/z_new_tests.log
G2M_RANK_WARP32=0 timeout 600 python -m pytest tests/test_gpu_round2.py -q -x -k "rank_copy" 2>&1 | tail -1
for v in 1 0; do G2M_RANK_WARP32=$v python scripts/e2e_debug.py cl4 > gpurun_out/z_e2e_cl4_w32_$v.txt 2>&1; echo "== w32=$v"; grep -h "plain\|orient degrees\|rank build" gpurun_out/z_e2e_cl4_w32_$v.txt | tail -6; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank|k_orient" -c 12 --csv --log-file gpurun_out/z_ncu_rank7.csv python scripts/e2e_debug.py cl4 > /dev/null 2>&1
