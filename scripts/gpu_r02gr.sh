# round 2: k = 5, d+ in (512, 1024]: rows in shared memory (24 warps) vs global/L1 (32 warps)
mkdir -p gpurun_out
timeout 1200 python scripts/ab_env.py 22 cl5 "G2M_CL5_GR=0|G2M_CL5_GR=1" debug > gpurun_out/cl5_gr_ab.txt 2>&1; echo ab rc=$?
grep -v "^\[g2m\]" gpurun_out/cl5_gr_ab.txt | tail -6
grep "launch 1:\|class 5" gpurun_out/cl5_gr_ab.txt
