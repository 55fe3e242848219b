# round 2: 4-cycle grid tier A/B (RED + sweep, range size, stage cap) at RMAT-25
mkdir -p gpurun_out
T=${1:-r02j}
timeout 600 python -m pytest tests -m gpu -q -x -k "cycle4" > gpurun_out/${T}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_pytest.log
AB_REPS=1 timeout 1800 python scripts/ab_env.py 25 c4 "G2M_C4_RED=0|G2M_C4_RED=1|G2M_C4_RED=1;G2M_C4_RANGE=8388608|G2M_C4_RED=1;G2M_C4_RANGE=33554432|G2M_C4_RED=1;G2M_C4_STAGE_CAP=67108864|G2M_C4_RED=1;G2M_C4_STAGE_CAP=4194304" debug > gpurun_out/${T}_c425_ab.txt 2>&1; echo c425 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c425_ab.txt
