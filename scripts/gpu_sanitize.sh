# compute-sanitizer memcheck / racecheck / synccheck on the small all-families workload
mkdir -p gpurun_out
T=${1:-r02s}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py ${2:-10} > gpurun_out/${T}_sanitize_${tool}.log 2>&1; echo $tool rc=$?; grep -E "ERROR SUMMARY|MISMATCHES|Error" gpurun_out/${T}_sanitize_${tool}.log | head -5
done
