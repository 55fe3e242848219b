# round 2 (z): rank-space rows: tiles (short rows) + warp register sort + CTA sort
mkdir -p gpurun_out
python scripts/e2e_debug.py cl4 > gpurun_out/z_e2e_cl4_v5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank|k_orient|tile" -c 30 --csv --log-file gpurun_out/z_ncu_rank5.csv python scripts/e2e_debug.py cl4 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -h "plain\|rank build" gpurun_out/z_e2e_cl4_v5.txt | tail -8
