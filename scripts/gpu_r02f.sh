# round 2: k=5 big-row phase (test + A/B), multi-GPU split simulations, 4-cycle tier
# breakdown at RMAT-25/27, then compute-sanitizer (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
T=${1:-r02f}
timeout 900 python -m pytest tests/test_gpu_round2.py -q -k "cl5_deferred or hub_core" > gpurun_out/${T}_pytest_new.log 2>&1; echo new tests rc=$?; tail -2 gpurun_out/${T}_pytest_new.log
AB_REPS=4 timeout 900 python scripts/ab_env.py 22 cl3,cl4 "G2M_PAIR_CORE=0|G2M_PAIR_CORE=14|G2M_PAIR_CORE=15|G2M_PAIR_CORE=16" debug > gpurun_out/${T}_core_ab.txt 2>&1; echo core ab rc=$?; grep -E "\] kernel|launch 4" gpurun_out/${T}_core_ab.txt
AB_REPS=3 timeout 900 python scripts/ab_env.py 22 cl5 "G2M_CL5_BIG=0|G2M_CL5_BIG=1" debug > gpurun_out/${T}_cl5_ab.txt 2>&1; echo cl5 ab rc=$?; grep -E "cl5 \[|launch" gpurun_out/${T}_cl5_ab.txt
for w in cl4 tc c4; do
  G2M_SIM_SPLITS=est:1,est:16,est:64,est:256,rr:1 timeout 1200 python bench.py --workload $w --steps 1 --warmup 1 --simulate-parts 8 --no-cpu-baseline --no-e2e --no-parity --no-roofline > gpurun_out/${T}_sim_${w}.json 2> gpurun_out/${T}_sim_${w}.err
  echo $w rc=$?; grep "simulated split" gpurun_out/${T}_sim_${w}.err
done
AB_REPS=1 timeout 900 python scripts/ab_env.py 25 c4 "X=0" debug > gpurun_out/${T}_c425_tiers.txt 2>&1; echo c425 rc=$?; grep -E "cycle4|c4 " gpurun_out/${T}_c425_tiers.txt | head -20
AB_REPS=1 timeout 1200 python scripts/ab_env.py 27 c4 "X=0" debug > gpurun_out/${T}_c427_tiers.txt 2>&1; echo c427 rc=$?; grep -E "cycle4|c4 " gpurun_out/${T}_c427_tiers.txt | head -20
