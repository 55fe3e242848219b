# round 2: sanitizers + focused ncu captures after the hub core (summarised on the box)
mkdir -p gpurun_out
T=${1:-r02q}
for tool in memcheck racecheck synccheck; do
  timeout 700 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py 10 > gpurun_out/${T}_sanitize_${tool}.log 2>&1; echo $tool rc=$?; grep -E "ERROR SUMMARY|MISMATCHES" gpurun_out/${T}_sanitize_${tool}.log | head -3
done
timeout 1200 bash scripts/gpu_r02m.sh r02m
