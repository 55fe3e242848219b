# N>1 bench path on one GPU: 2 ranks (gloo collectives) folded onto cuda:0; counts must equal N=1
set -x
for w in cl4 tc c4; do
  G2M_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $w --scale 18 --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N2', d['config']['workload'], d['counts'], d['n_gpus'], d['e2e']['value'] is not None, d['roofline']['algorithmic_bytes_per_step'])"
  timeout 600 python bench.py --workload $w --scale 18 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1', d['config']['workload'], d['counts'], d['roofline']['algorithmic_bytes_per_step'])"
done
G2M_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --scale 18 --steps 1 --warmup 1 2>&1 | tail -2 | cut -c1-200
