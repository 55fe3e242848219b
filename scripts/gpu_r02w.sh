# e2e investigation: TC / 4-clique public-API calls, phase split, with G2M_DEBUG phases
mkdir -p gpurun_out
T=${1:-r02w}
timeout 600 python scripts/e2e_breakdown.py tc > gpurun_out/${T}_e2e_tc.txt 2>&1; echo tc rc=$?; cat gpurun_out/${T}_e2e_tc.txt | tail -4
G2M_DEBUG=1 timeout 600 python scripts/e2e_breakdown.py tc > gpurun_out/${T}_e2e_tc_dbg.txt 2>&1; echo tcdbg rc=$?; grep -E "rank build|orient|core|^[0-9]" gpurun_out/${T}_e2e_tc_dbg.txt | tail -30
