# round 2: ncu --set full of the preprocessing kernels of one public-API 4-clique call (RMAT-22)
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_orient_keep_tiles|k_orient_fill_slots|k_rank_fill|k_rank_classify" -c 7 \
  -o /tmp/ncu/pre -f python scripts/e2e_debug.py cl4 > /dev/null 2> /tmp/ncu/pre.err; echo ncu rc=$?
python scripts/profile_summary.py /tmp/ncu/pre.ncu-rep "preprocess@rmat22" gpurun_out/r02z_preprocess_ncu.md > /dev/null 2>&1; echo summary rc=$?
cat gpurun_out/r02z_preprocess_ncu.md
