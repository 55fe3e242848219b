# round 2: hub-core CTA rows + c4 run aggregation + generated-kernel occupancy, tests and A/B
mkdir -p gpurun_out
T=${1:-r02h}
timeout 900 python -m pytest tests -m gpu -q -x -k "hub_core or cycle4 or c4 or grid or lgs_clique or clique_kernels or rmat12" > gpurun_out/${T}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_pytest.log
AB_REPS=4 timeout 900 python scripts/ab_env.py 22 cl3,cl4,cl5 "G2M_CTA_CORE=0|G2M_CTA_CORE=1|G2M_CTA_CORE=1;G2M_PAIR_CORE=17" debug > gpurun_out/${T}_ctacore_ab.txt 2>&1; echo ctacore rc=$?; grep -E "\] kernel" gpurun_out/${T}_ctacore_ab.txt
AB_REPS=2 timeout 900 python scripts/ab_env.py 27 cl3 "G2M_CTA_CORE=0|G2M_CTA_CORE=1" debug > gpurun_out/${T}_tc27_ab.txt 2>&1; echo tc27 rc=$?; grep -E "\] kernel|launch" gpurun_out/${T}_tc27_ab.txt
AB_REPS=2 timeout 900 python scripts/ab_env.py 24 c4 "X=0" debug > gpurun_out/${T}_c4_ab.txt 2>&1; echo c4 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c4_ab.txt | head -12
for sw in "4096 1024" "0 1024" "0 256"; do
  set -- $sw
  G2M_SMEM_SLOT_WORDS=$1 G2M_STAGE_WORDS=$2 timeout 300 python bench.py --workload mc4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-roofline --no-parity > gpurun_out/${T}_mc4_$1_$2.json 2> /dev/null
  echo mc4 slots=$1 stage=$2 $(python scripts/line_summary.py gpurun_out/${T}_mc4_$1_$2.json | cut -c1-120)
done
