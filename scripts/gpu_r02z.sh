# round 2 (z): slot-parallel orientation; rank-row CTA threshold A/B
mkdir -p gpurun_out
for m in 128 64 32; do
  G2M_RANK_MID=$m python scripts/e2e_debug.py cl4 > gpurun_out/z_e2e_cl4_mid$m.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for m in 128 64 32; do echo "== mid $m"; grep -h "plain\|orient\|rank build" gpurun_out/z_e2e_cl4_mid$m.txt | tail -12; done
