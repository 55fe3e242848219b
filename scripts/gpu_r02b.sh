# round 2: 4-cycle grid-tier fix check + clique tier launch-mode A/B
mkdir -p gpurun_out
T=${1:-r02b}
timeout 600 python -m pytest tests -m gpu -x -q -k "cycle4 or grid or concurrent" > gpurun_out/${T}_pytest_c4.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${T}_pytest_c4.log
timeout 900 python scripts/ab_tiers.py 22 3,4,5 8,1,2,4 > gpurun_out/${T}_ab.txt 2> gpurun_out/${T}_ab.err; echo ab rc=$?; cat gpurun_out/${T}_ab.txt; grep "launch\|class\|buckets" gpurun_out/${T}_ab.err | head -60
