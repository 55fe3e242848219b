# round 2 final sweep, part 2: config C5 on device-generated R-MAT (TC RMAT-27, 4-cycle RMAT-25/27)
mkdir -p gpurun_out
T=${1:-r02l}
run() { n=$1; lim=$2; shift; shift; timeout $lim python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err; echo $n rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_$n.json | cut -c1-300; }
run tc27 700 --workload tc --scale 27 --steps 3 --warmup 3
run c425 600 --workload c4 --scale 25 --steps 2 --warmup 3
run c427 1500 --workload c4 --scale 27 --steps 2 --warmup 3 --balg-sample 1e-5 --cpu-seconds 20
# the 8-part split simulation with the final kernels (estimator defaults), and the N=2 path folded onto one GPU
G2M_SIM_SPLITS=est:16,rr:1 timeout 600 python bench.py --workload cl4 --steps 1 --warmup 1 --simulate-parts 8 --no-cpu-baseline --no-e2e --no-parity --no-roofline > gpurun_out/${T}_sim_cl4.json 2> gpurun_out/${T}_sim_cl4.err; echo sim rc=$?; grep "simulated split" gpurun_out/${T}_sim_cl4.err
G2M_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --workload cl4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_cl4_n2gloo.json 2> gpurun_out/${T}_bench_cl4_n2gloo.err; echo n2 rc=$?; python scripts/line_summary.py gpurun_out/${T}_bench_cl4_n2gloo.json | cut -c1-250
