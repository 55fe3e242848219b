# round 2: tier breakdowns after the hub-core change (cl3/cl4/cl5 RMAT-22), 4-cycle wedge bounds per tier,
# generated-kernel defaults on the motif configs
mkdir -p gpurun_out
T=${1:-r02i}
AB_REPS=2 timeout 600 python scripts/ab_env.py 22 cl3,cl4,cl5 "X=0" debug > gpurun_out/${T}_cl_tiers.txt 2>&1; echo cl rc=$?; grep -E "\] kernel|launch|buckets" gpurun_out/${T}_cl_tiers.txt
AB_REPS=1 timeout 900 python scripts/ab_env.py 25 c4 "X=0" debug > gpurun_out/${T}_c425.txt 2>&1; echo c425 rc=$?; grep -E "c4 \[|cycle4" gpurun_out/${T}_c425.txt | head
for w in mc3 mc4; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-roofline > gpurun_out/${T}_$w.json 2> /dev/null; echo $w $(python scripts/line_summary.py gpurun_out/${T}_$w.json | cut -c1-220)
done
