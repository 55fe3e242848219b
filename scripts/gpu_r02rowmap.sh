# round 2: tile row map, block passes (0) vs per-warp segments carried by a segment-max pass (1)
mkdir -p gpurun_out
for v in 0 1; do
  G2M_ROWMAP=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank_fill_tiles" -c 3 --csv --log-file gpurun_out/rowmap_ncu_$v.csv python scripts/e2e_debug.py cl4 > /dev/null 2>&1
  echo "== rowmap $v"; grep duration gpurun_out/rowmap_ncu_$v.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,150-
done
