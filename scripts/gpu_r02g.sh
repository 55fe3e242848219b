# round 2 ncu sweep (summaries built on the box)
bash scripts/gpu_ncu_r02.sh ${1:-r02n} "${2:-cl4 tc cl5 tc:G2M_PAIR_BULK=1 c4 diamond mc3 mc4 tc27}"
