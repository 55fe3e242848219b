# e2e phase breakdown of one public-API call (upload, orientation, rank build, kernels)
mkdir -p gpurun_out
T=${1:-e2e}
for w in ${2:-cl4 tc}; do
  G2M_DEBUG=1 timeout 600 python scripts/e2e_breakdown.py $w > gpurun_out/${T}_$w.log 2>&1; echo $w rc=$?
  grep -v "launch [0-9]" gpurun_out/${T}_$w.log | tail -40
done
