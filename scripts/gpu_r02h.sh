# round 2: generated-kernel occupancy A/B (shared vs global slots) on the motif configs,
# c4 run-aggregated staging check + timing
mkdir -p gpurun_out
T=${1:-r02h}
timeout 900 python -m pytest tests -m gpu -q -x -k "cycle4 or c4 or grid" > gpurun_out/${T}_pytest_c4.log 2>&1; echo c4 tests rc=$?; tail -2 gpurun_out/${T}_pytest_c4.log
for sw in "4096 1024" "0 1024" "0 256" "2048 512"; do
  set -- $sw
  G2M_SMEM_SLOT_WORDS=$1 G2M_STAGE_WORDS=$2 timeout 600 python bench.py --workload mc4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-roofline --no-parity > gpurun_out/${T}_mc4_$1_$2.json 2> /dev/null
  echo mc4 slots=$1 stage=$2 $(python scripts/line_summary.py gpurun_out/${T}_mc4_$1_$2.json | cut -c1-160)
  G2M_SMEM_SLOT_WORDS=$1 G2M_STAGE_WORDS=$2 timeout 600 python bench.py --workload mc3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-roofline --no-parity > gpurun_out/${T}_mc3_$1_$2.json 2> /dev/null
  echo mc3 slots=$1 stage=$2 $(python scripts/line_summary.py gpurun_out/${T}_mc3_$1_$2.json | cut -c1-160)
done
AB_REPS=3 timeout 900 python scripts/ab_env.py 24 c4 "X=0" debug > gpurun_out/${T}_c4_ab.txt 2>&1; echo c4 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c4_ab.txt | head -12
