mkdir -p gpurun_out
python scripts/e2e_breakdown.py cl4 > gpurun_out/z_e2e_breakdown_cl4.txt 2>&1
G2M_DEBUG=1 python scripts/e2e_debug.py cl4 > gpurun_out/z_e2e_debug_cl4b.txt 2>&1
python scripts/e2e_breakdown.py tc > gpurun_out/z_e2e_breakdown_tc.txt 2>&1
cat gpurun_out/z_e2e_breakdown_cl4.txt gpurun_out/z_e2e_breakdown_tc.txt; grep -v "launch\|class" gpurun_out/z_e2e_debug_cl4b.txt | tail -14
