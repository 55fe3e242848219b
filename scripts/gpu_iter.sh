# quick iteration: parity subset + benches of the clique path
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "lgs or rmat12 or clique or golden" 2>&1 | tail -5
G2M_DEBUG=1 timeout 600 python bench.py --workload cl4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-roofline 2>&1 | grep -E "launch|^\{|class|buckets" | tail -22
G2M_TC_LGS=1 G2M_DEBUG=1 timeout 600 python bench.py --workload tc --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-roofline 2>&1 | grep -E "launch|^\{|class|buckets" | tail -22
G2M_DEBUG=1 timeout 600 python bench.py --workload cl5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-roofline 2>&1 | grep -E "launch|^\{|class|buckets" | tail -22
