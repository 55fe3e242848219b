# round 2: heaviest-first source order inside the CTA tiers (G2M_CLIQUE_LPT) A/B, RMAT-22 k = 3, 4, 5
mkdir -p gpurun_out
timeout 1200 python scripts/ab_env.py 22 cl3,cl4,cl5 "G2M_CLIQUE_LPT=0|G2M_CLIQUE_LPT=1" debug > gpurun_out/lpt_ab.txt 2>&1; echo ab rc=$?
grep -v "^\[g2m\]" gpurun_out/lpt_ab.txt | tail -12
grep "launch" gpurun_out/lpt_ab.txt
