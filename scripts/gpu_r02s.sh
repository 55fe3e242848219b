# round 2: pair-tier loads-in-flight A/B; e2e breakdown of the 5-clique public-API call
mkdir -p gpurun_out
T=${1:-r02s}
AB_REPS=4 timeout 900 python scripts/ab_env.py 22 cl3,cl4 "G2M_PAIR_PU=1|G2M_PAIR_PU=2|G2M_PAIR_PU=4" debug > gpurun_out/${T}_pu.txt 2>&1; echo pu rc=$?; grep -E "\] kernel|launch 4" gpurun_out/${T}_pu.txt
timeout 600 python scripts/e2e_breakdown.py cl5 > gpurun_out/${T}_e2e_cl5.txt 2>&1; echo e2e rc=$?; tail -4 gpurun_out/${T}_e2e_cl5.txt
timeout 600 python scripts/e2e_breakdown.py cl4 > gpurun_out/${T}_e2e_cl4.txt 2>&1; echo e2e rc=$?; tail -3 gpurun_out/${T}_e2e_cl4.txt
