# one default bench run (+ optional extra args), output to gpurun_out/<tag>.json/.err
TAG=${1:-bench}; shift
timeout 1500 python bench.py "$@" > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err; echo rc=$?
cat gpurun_out/${TAG}.json; tail -15 gpurun_out/${TAG}.err
