# round 2 (z): k = 5 heavy rows counted word-outer (G2M_CL5_Q=1) vs lane-per-l (0); e2e phases of diamond after the max-degree fix
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py 22 cl5 "G2M_CL5_Q=0|G2M_CL5_Q=1" debug > gpurun_out/z_cl5_q_ab.txt 2>&1; echo ab rc=$?
grep -v "^\[g2m\]   launch" gpurun_out/z_cl5_q_ab.txt | grep -v "class" | tail -12
grep "launch 1:" gpurun_out/z_cl5_q_ab.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/e2e_profile.py diamond > gpurun_out/z_prof_diamond.txt 2>&1; grep "api ms" gpurun_out/z_prof_diamond.txt
