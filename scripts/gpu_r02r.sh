# round 2: batched hub-core reads (tests + timing)
mkdir -p gpurun_out
T=${1:-r02r}
timeout 900 python -m pytest tests -m gpu -q -x -k "hub_core or clique or lgs or staged_pair" > gpurun_out/${T}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_pytest.log
AB_REPS=4 timeout 900 python scripts/ab_env.py 22 cl3,cl4,cl5 "X=0" debug > gpurun_out/${T}_cl.txt 2>&1; echo cl rc=$?; grep -E "\] kernel|launch" gpurun_out/${T}_cl.txt
AB_REPS=2 timeout 900 python scripts/ab_env.py 27 cl3 "X=0" > gpurun_out/${T}_tc27.txt 2>&1; echo tc27 rc=$?; grep -E "\] kernel" gpurun_out/${T}_tc27.txt
