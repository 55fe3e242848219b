"""Multi-process path on CPU (gloo, world size 2): the chunked round-robin
shares that bench.py / run_on_devices hand to each GPU partition the task
list, per-rank counts add up to the whole count, and the 128-bit count
reduction is exact. The per-rank mining here is the CPU oracle (test
infrastructure); on GPUs it is the same share run by the kernels."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import graphs as G
from oracle import oracle as O
from paper_2112_09761_b200 import distributed as D
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import plan as PL
from paper_2112_09761_b200 import scheduler
from util import cycle4, diamond, make_plan, orient_host

from paper_2112_09761_b200 import pattern as P


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _edge_tasks(g):
    off = np.asarray(g.row_offsets, dtype=np.int64)
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(off))
    return np.column_stack([src, g.neighbors.astype(np.int64)])


def _worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        chunk, parts, part = D.shard(rank, world, chunk=16)
        g = GR.from_edges(G.rmat_edges(10, 8, 3), num_vertices=1 << 10)
        out = {}
        # edge-task share (generated plan kernels): implicit list, chunked RR
        for name, gg, f in [
            ("diamond", g, PL.as_forest(make_plan(diamond(), g, rewrite=True))),
            ("4-cycle", g, PL.as_forest(make_plan(cycle4(), g))),
        ]:
            all_t = _edge_tasks(gg)
            q = scheduler.split_chunked_rr(np.arange(len(all_t)), parts, 1, alpha=chunk).queues[part]
            mine, _ = O.run(gg, f, tasks=all_t[q], edge=True)
            out[name] = D.allreduce_counts(mine)
        # source-vertex share (LGS clique / wedge kernels): (v // chunk) % parts == part
        og = orient_host(g)
        f4 = PL.as_forest(make_plan(P.generate_clique(4), g, oriented=True))
        all_t = _edge_tasks(og)
        keep = (all_t[:, 0] // chunk) % parts == part
        mine, _ = O.run(og, f4, tasks=all_t[keep], edge=True)
        out["4-clique"] = D.allreduce_counts(mine)
        # exact 128-bit reduction
        out["big"] = D.allreduce_counts({"a": (1 << 100) + rank, "b": (1 << 64) - 1, "c": 0})
        out["max"] = D.allreduce_max(1.5 + rank)
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_and_reduction():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert set(results.keys()) == {0, 1}
    g = GR.from_edges(G.rmat_edges(10, 8, 3), num_vertices=1 << 10)
    want = {
        "diamond": O.run(g, PL.as_forest(make_plan(diamond(), g, rewrite=True)))[0],
        "4-cycle": O.run(g, PL.as_forest(make_plan(cycle4(), g)))[0],
        "4-clique": O.run(orient_host(g), PL.as_forest(make_plan(P.generate_clique(4), g,
                                                                  oriented=True)))[0],
    }
    for r in range(world):
        res = results[r]
        for k, v in want.items():
            assert res[k] == v, (r, k)
        assert res["big"] == {"a": (1 << 101) + 1, "b": 2 * ((1 << 64) - 1), "c": 0}
        assert res["max"] == 2.5


def test_shard_and_limbs():
    assert D.shard(0, 1) is None
    assert D.shard(3, 8, chunk=256) == (256, 8, 3)
    # c = alpha * y: alpha = 2, y = resident warps
    assert D.shard(3, 8) == (D.ALPHA * D.resident_warps(), 8, 3)
    assert D.resident_warps() > 0
    with pytest.raises(ValueError):
        D.shard(8, 8)
    for v in (0, 1, (1 << 32) - 1, 1 << 64, (1 << 128) - 1):
        assert D.from_limbs(D.to_limbs(v)) == v
    with pytest.raises(ValueError):
        D.to_limbs(1 << 128)


def test_source_spec_fields():
    from paper_2112_09761_b200 import executor as EX
    s = EX.source_spec(None)
    assert s.rr_chunk == 0 and s.weighted == 0
    s = EX.source_spec((18944, 8, 3))
    assert (s.rr_chunk, s.weighted, s.rr_parts, s.rr_part) == (EX.SOURCE_CHUNK["lgs"], 1, 8, 3)
    s = EX.source_spec((18944, 8, 3), family="cycle4")
    assert s.rr_chunk == EX.SOURCE_CHUNK["cycle4"]
    s = EX.source_spec((18944, 8, 3), "rr", 1)
    assert (s.rr_chunk, s.weighted, s.rr_parts, s.rr_part) == (1, 0, 8, 3)
    with pytest.raises(ValueError):
        EX.source_spec((1, 2, 0), "bogus")


def test_bench_gpus_mismatch_exits_nonzero():
    import subprocess
    import sys
    from pathlib import Path
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(Path(__file__).resolve().parent.parent / "bench.py"),
                          "--gpus", "2"], capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stdout


def _support_share(og, chunk, parts, part):
    """Host restatement of one rank's g2m_diamond_support: triangles whose DAG
    source u has (u // chunk) % parts == part add 1 to the support of each of
    their three DAG edges (indexed by oriented slot)."""
    off = np.asarray(og.row_offsets, dtype=np.int64)
    nbr = og.neighbors.astype(np.int64)
    t = np.zeros(len(nbr), dtype=np.int32)
    slot = {}
    for u in range(og.num_vertices):
        for s in range(off[u], off[u + 1]):
            slot[(u, int(nbr[s]))] = s
    for u in range(og.num_vertices):
        if parts > 1 and (u // chunk) % parts != part:
            continue
        nu = nbr[off[u]:off[u + 1]]
        for i, v in enumerate(nu):
            for w in nu[i + 1:]:
                for a, b in ((v, w), (w, v)):
                    s = slot.get((int(a), int(b)))
                    if s is not None:   # triangle u, v, w
                        t[slot[(u, int(v))]] += 1
                        t[slot[(u, int(w))]] += 1
                        t[s] += 1
    return t


def _support_worker(rank, world, port, results):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = GR.from_edges(G.rmat_edges(9, 8, 5), num_vertices=1 << 9)
        og = orient_host(g)
        t = torch.from_numpy(_support_share(og, 4, world, rank))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)            # the one data-path collective
        n = len(t)
        mine = t[rank * n // world:(rank + 1) * n // world].to(torch.int64)
        share = int((mine * (mine - 1) // 2).sum())
        results[rank] = (D.allreduce_counts({"diamond": share}), t.numpy().tolist())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_diamond_support_allreduce():
    """The multi-GPU diamond protocol (distributed.diamond_count) with the
    kernels restated on the host: support shares by source, all-reduce of the
    support array, C(t, 2) over slot shares, count reduction; equals the
    oracle's diamond count and the unsplit support."""
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_support_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    g = GR.from_edges(G.rmat_edges(9, 8, 5), num_vertices=1 << 9)
    want = O.run(g, PL.as_forest(make_plan(diamond(), g, rewrite=True)))[0]
    full = _support_share(orient_host(g), 4, 1, 0).tolist()
    for r in range(world):
        counts, t = results[r]
        assert counts == want
        assert t == full
