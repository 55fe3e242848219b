# staged pair tier A/B (+ test), then ncu evidence for every config
mkdir -p gpurun_out
T=${1:-r02d}
timeout 600 python -m pytest tests -m gpu -x -q -k "staged_pair or concurrent or gcsr" > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python scripts/ab_env.py 22 cl3,cl4,cl5 "G2M_PAIR_BULK=0|G2M_PAIR_BULK=1|G2M_PAIR_BULK=2" debug > gpurun_out/${T}_ab.txt 2> gpurun_out/${T}_ab.err; echo ab rc=$?; cat gpurun_out/${T}_ab.txt; grep -i "pair\|launch 4\|launch 5" gpurun_out/${T}_ab.err
bash scripts/gpu_ncu_r02.sh r02n "cl4 tc cl5 c4 diamond mc3 mc4"
