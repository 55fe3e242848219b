# configs 3/4 at reduced and full scale (timeouts bound each)
for spec in "c4 --scale 20" "diamond --scale 20" "c4 --scale 22" "diamond --scale 24" "mc3" "mc4" "mc4 --n 20000"; do
  echo "=== $spec"
  G2M_DEBUG=1 timeout 400 python bench.py --workload $spec --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "^\{|algorithmic|Error|error" | cut -c1-700
done
