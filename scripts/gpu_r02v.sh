# round 2: 4-cycle grid-staged tier (tests + A/B RMAT-25, RMAT-27)
mkdir -p gpurun_out
T=${1:-r02v}
timeout 600 python -m pytest tests -m gpu -q -x -k "cycle4" > gpurun_out/${T}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_pytest.log
AB_REPS=1 timeout 900 python scripts/ab_env.py 25 c4 "G2M_C4_GSTAGE=0|G2M_C4_GSTAGE=1" debug > gpurun_out/${T}_c425.txt 2>&1; echo c425 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c425.txt | head -14
AB_REPS=1 timeout 1200 python scripts/ab_env.py 27 c4 "G2M_C4_GSTAGE=1" debug > gpurun_out/${T}_c427.txt 2>&1; echo c427 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c427.txt | head -8
