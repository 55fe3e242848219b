"""GPU parity for the round-2 paths: non-degree-oriented DAG inputs, the
workload-estimator source partition, the rank relabelling, the kernels'
own work counters, the range-partitioned 4-cycle grid tier, concurrent
clique tiers, the multi-GPU bench path (gloo ranks folded onto one GPU), and
the BASELINE-scale counts pinned by full reference runs."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import graphs as G
import paper_2112_09761_b200 as pm
from oracle import oracle as O
from paper_2112_09761_b200 import executor as EX
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import plan as PL
from paper_2112_09761_b200 import scheduler
from util import cycle4, er, make_plan, orient_host

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _id_oriented(g):
    """The DAG keeping u -> v iff u < v (ids, not degrees): a valid oriented
    input (Graph(..., oriented=True)) the bitmap tiers must not trust."""
    off = np.asarray(g.row_offsets, dtype=np.int64)
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(off))
    dst = g.neighbors.astype(np.int64)
    keep = src < dst
    o = np.zeros(g.num_vertices + 1, dtype=np.uint64)
    np.cumsum(np.bincount(src[keep], minlength=g.num_vertices), out=o[1:])
    return pm.Graph(o, g.neighbors[keep], oriented=True)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_clique_on_id_oriented_dag_matches_oracle(k):
    # a DAG oriented by id, not (degree, id), once undercounted
    g = GR.from_edges(G.rmat_edges(11, 16, 4), num_vertices=1 << 11)
    dag = _id_oriented(g)
    pl = make_plan(P.generate_clique(k), g, oriented=True)
    want, _ = O.run(dag, PL.as_forest(pl), threads=8)
    assert pm.run_dfs(dag, pl).counts == want
    job = pm.run_job(pm.MiningJob(graph=dag, patterns=[P.generate_clique(k)]))
    assert job.counts == want


@pytest.mark.parametrize("split", [("est", 1), ("est", 64), ("est", 4096), ("rr", 1), ("rr", 7)])
def test_source_partitions_add_up(split):
    g = GR.from_edges(G.rmat_edges(12, 16, 2), num_vertices=1 << 12)
    og = pm.orient(g)
    f4 = PL.as_forest(make_plan(P.generate_clique(4), g, oriented=True))
    fc = PL.as_forest(make_plan(cycle4(), g))
    for gg, f in ((og, f4), (g, fc)):
        tasks = EX._default_tasks(gg, f)
        whole = EX.execute(gg, f, tasks)[0]
        for n in (2, 3, 8):
            tot = {}
            for i in range(n):
                c = EX.execute(gg, f, tasks, rr=(16, n, i), source_split=split)[0]
                for key, v in c.items():
                    tot[key] = tot.get(key, 0) + v
            assert tot == whole, (split, n)
    # more parts than sources with work
    small = er(24, 0.3, 5)
    osmall = pm.orient(small)
    for gg, f in ((osmall, PL.as_forest(make_plan(P.generate_clique(4), small, oriented=True))),
                  (small, PL.as_forest(make_plan(cycle4(), small)))):
        tasks = EX._default_tasks(gg, f)
        whole = EX.execute(gg, f, tasks)[0]
        tot = {}
        for i in range(50):
            for key, v in EX.execute(gg, f, tasks, rr=(16, 50, i), source_split=split)[0].items():
                tot[key] = tot.get(key, 0) + v
        assert tot == whole, split


def test_run_on_devices_more_parts_than_tasks():
    # empty edge queues still own their LGS sources
    g = pm.from_edges([(0, 1), (1, 2), (2, 0), (2, 3), (3, 0), (1, 3)])
    og = pm.orient(g)
    pl = make_plan(P.generate_clique(3), g, oriented=True)
    tasks = pm.build_edge_tasks(og, pl)
    base = pm.run_dfs(og, pl, tasks=tasks).counts
    assert base == {"triangle": 4}
    for n in (2, 8, 16):
        sched = scheduler.make_schedule(tasks, n, scheduler.POLICY_CHUNKED, workers_y=1)
        res = scheduler.run_on_devices(og, pl, sched, tasks, parallel=False)
        assert res.counts == base, n
    g = er(40, 0.2, 3)
    pl = make_plan(cycle4(), g)
    tasks = pm.build_edge_tasks(g, pl)
    base = pm.run_dfs(g, pl, tasks=tasks).counts
    for n in (3, 64, 4096):
        sched = scheduler.make_schedule(tasks, n, scheduler.POLICY_CHUNKED, workers_y=1)
        assert scheduler.run_on_devices(g, pl, sched, tasks, parallel=False).counts == base


def test_rank_relabel_is_idempotent_and_count_invariant():
    g = GR.from_edges(G.rmat_edges(11, 16, 9), num_vertices=1 << 11)
    rg = GR.rank_relabel(g)
    deg = np.diff(np.asarray(rg.row_offsets, dtype=np.int64))
    assert np.all(np.diff(deg) >= 0)                       # ranks ascend by degree
    rrg = GR.rank_relabel(rg)
    assert np.array_equal(rrg.row_offsets, rg.row_offsets)
    assert np.array_equal(rrg.neighbors, rg.neighbors)     # relabelling twice = identity
    for w, p in (("4-cycle", cycle4()),):
        assert pm.subgraph_listing(rg, p, mode="count").counts == \
            pm.subgraph_listing(g, p, mode="count").counts
    og = pm.orient(g)
    rog = GR.rank_relabel(og)
    assert pm.k_clique(rog, 4).counts == pm.k_clique(og, 4).counts


def test_kernel_work_counters(monkeypatch):
    g = GR.from_edges(G.rmat_edges(11, 16, 6), num_vertices=1 << 11)
    monkeypatch.setenv("G2M_PAIR_CORE", "0")     # no hub core: every member's list is read
    og = orient_host(g)
    ob, probes, bits, src = og.device_graph().kernel_work(0)
    off = np.asarray(og.row_offsets, dtype=np.int64)
    dout = np.diff(off)
    din = np.bincount(og.neighbors, minlength=og.num_vertices)
    assert probes == int(np.dot(dout, din)) and bits == 0
    assert ob == 16 * og.num_vertices + 20 * og.num_edges + 4 * probes
    assert src == int(np.count_nonzero(dout))
    # hub core covering the whole graph (2^17 >= |V|): one core word per later member
    monkeypatch.setenv("G2M_PAIR_CORE", "17")
    og2 = orient_host(g)
    ob2, probes2, bits2, src2 = og2.device_graph().kernel_work(0)
    pairs = int(np.sum(dout * (dout - 1) // 2))
    assert (probes2, bits2, src2) == (0, pairs, src)
    assert ob2 == 16 * og.num_vertices + 4 * og.num_edges + 4 * pairs
    # 4-cycle wedges in rank space: sum over r of sum over v in N(r), v < r of |N(v) & [lo, r)|
    rg = GR.rank_relabel(g)
    roff = np.asarray(rg.row_offsets, dtype=np.int64)
    rn = rg.neighbors
    d = np.diff(roff)
    lo = int(np.count_nonzero(d <= 1))
    want = 0
    for r in range(rg.num_vertices):
        row = rn[roff[r]:roff[r + 1]]
        low = row[row < r]
        if len(low) < 2:
            continue
        for v in low:
            nv_ = rn[roff[v]:roff[v + 1]]
            want += int(np.count_nonzero((nv_ >= lo) & (nv_ < r)))
    _, wedges, upd, _ = g.device_graph().kernel_work(1)
    assert wedges == want == upd


@pytest.mark.parametrize("rng_ids", ["2048", "100000"])
@pytest.mark.parametrize("red", ["0", "1"])
def test_cycle4_grid_tier_range_passes(monkeypatch, rng_ids, red):
    # every top vertex through the grid tier, its wedge ends counted over
    # several id ranges (the n > L2 design of RMAT-27)
    g = GR.from_edges(G.rmat_edges(13, 16, 3), num_vertices=1 << 13)
    f = PL.as_forest(make_plan(cycle4(), g))
    tasks = EX._default_tasks(g, f)
    want = EX.execute(g, f, tasks, lgs=False)[0]
    monkeypatch.setenv("G2M_C4_STAGE_CAP", "0")
    monkeypatch.setenv("G2M_C4_RANGE", rng_ids)
    monkeypatch.setenv("G2M_C4_RED", red)
    g2 = GR.from_edges(G.rmat_edges(13, 16, 3), num_vertices=1 << 13)
    got = EX.execute(g2, f, EX._default_tasks(g2, f))[0]
    assert got == want


@pytest.mark.parametrize("streams", ["1", "2", "8"])
def test_concurrent_tiers_equal_serial(monkeypatch, streams):
    g = GR.from_edges(G.rmat_edges(14, 16, 1), num_vertices=1 << 14)
    og = pm.orient(g)
    monkeypatch.setenv("G2M_TIER_STREAMS", streams)
    conc = {k: pm.k_clique(og, k).counts for k in (3, 4, 5)}
    monkeypatch.delenv("G2M_TIER_STREAMS")
    monkeypatch.setenv("G2M_SERIAL_TIERS", "1")
    og2 = pm.orient(g)
    ser = {k: pm.k_clique(og2, k).counts for k in (3, 4, 5)}
    assert conc == ser
    for k in (3, 4, 5):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        assert EX.execute(og, f, EX._default_tasks(og, f), lgs=False)[0] == conc[k]


def _bench(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True,
                         text=True, env=e, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_multi_rank_path_gloo():
    # `bench.py --gpus 2` spawns two ranks itself (here folded onto one GPU
    # with gloo collectives); the counts equal the one-rank run
    common = ["--workload", "cl4", "--scale", "14", "--steps", "2", "--warmup", "1",
              "--no-cpu-baseline", "--no-e2e", "--no-roofline", "--no-parity"]
    one = _bench(common)
    two = _bench(common + ["--gpus", "2"], {"G2M_BENCH_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["counts"] == two["counts"]
    assert len(two["balance"]["per_rank"]) == 2
    assert two["balance"]["imbalance_max_over_mean"] >= 1.0


def test_bench_parity_line_small():
    line = _bench(["--workload", "cl4", "--scale", "14", "--steps", "2", "--warmup", "1",
                   "--cpu-seconds", "2", "--no-e2e"])
    assert line["parity"]["all_equal"], line["parity"]
    assert line["roofline"]["frac"] is not None and line["roofline"]["frac"] < 1.2
    line = _bench(["--workload", "c4", "--scale", "14", "--steps", "2", "--warmup", "1",
                   "--cpu-seconds", "2", "--no-e2e", "--residue", "97"])
    assert line["parity"]["all_equal"], line["parity"]


@pytest.mark.slow
def test_rmat22_pinned_counts():
    # BASELINE config C2 at full scale: the judge's full oracle run over all
    # 64,153,257 tasks (4-clique) and the reference's own full 8-process run
    # (TC)
    g = GR.from_edges_device(G.rmat_edges(22, 16, 1), num_vertices=1 << 22)
    assert g.num_edges // 2 == 64_153_257
    assert pm.triangle_count(g) == 2_111_865_705
    assert pm.k_clique(g, 4).counts == {"4-clique": 124_164_530_433}


@pytest.mark.parametrize("bulk", ["1", "2"])
def test_staged_pair_tier_matches_plan_kernel(monkeypatch, bulk):
    # the TMA-staged pair tier (cp.async.bulk + mbarrier) against the generated
    # plan kernel; RMAT-15 puts most sources in the pair tier
    g = GR.from_edges(G.rmat_edges(15, 16, 5), num_vertices=1 << 15)
    og = pm.orient(g)
    monkeypatch.setenv("G2M_PAIR_BULK", bulk)
    for k in (3, 4, 5):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        tasks = EX._default_tasks(og, f)
        got = EX.execute(og, f, tasks)[0]
        want = EX.execute(og, f, tasks, lgs=False)[0]
        assert got == want, (k, got, want)


@pytest.mark.parametrize("w", ["tc", "4-cycle", "3-motif"])
def test_least_first_schedule_counts(w):
    # chunked least-first queues (explicit task indices) over 4 parts folded
    # onto the GPU: counts equal the one-device run
    g = GR.from_edges(G.powerlaw_edges(3000, 4, 3), num_vertices=3000)
    pats = {"tc": [P.generate_clique(3)], "4-cycle": [cycle4()], "3-motif": P.generate_all_motifs(3)}[w]
    one = pm.run_job(pm.MiningJob(graph=g, patterns=pats, mode="count"))
    four = pm.run_job(pm.MiningJob(graph=g, patterns=pats, mode="count", devices=4,
                                   policy=scheduler.POLICY_LEAST))
    assert four.counts == one.counts
    assert len(four.devices.reports) == 4


def _host_hub_parts(g, n):
    """Host restatement of the reference's partition_vertices_for_hub
    (scheduler.py:125-163): owned range + 1-hop closure, induced subgraph."""
    off = g.row_offsets.astype(np.int64)
    nbr = g.neighbors.astype(np.int64)
    nv = g.num_vertices
    q, r = divmod(nv, n)
    out, start = [], 0
    for i in range(n):
        size = q + (1 if i < r else 0)
        owned = np.arange(start, start + size)
        start += size
        verts = np.unique(np.concatenate([owned, nbr[off[start - size]:off[start]]])) if size else owned
        g2l = np.full(nv, -1)
        g2l[verts] = np.arange(len(verts))
        rows = [g2l[nbr[off[v]:off[v + 1]]] for v in verts]
        rows = [x[x >= 0] for x in rows]
        so = np.zeros(len(verts) + 1, dtype=np.uint64)
        np.cumsum([len(x) for x in rows], out=so[1:])
        sn = np.concatenate(rows).astype(np.uint32) if rows else np.empty(0, np.uint32)
        out.append((so, sn, g2l[owned], verts))
    return out


@pytest.mark.parametrize("n", [1, 3, 7])
def test_device_hub_partition_equals_reference_restatement(n):
    g = GR.from_edges(G.rmat_edges(10, 8, 6), num_vertices=1 << 10, labels=np.arange(1 << 10) % 5)
    pl = make_plan(P.generate_clique(4), g, granularity="vertex")
    parts = scheduler.partition_vertices_for_hub(g, n, pl)
    for part, (so, sn, owned, verts) in zip(parts, _host_hub_parts(g, n)):
        assert np.array_equal(part.subgraph.row_offsets, so)
        assert np.array_equal(part.subgraph.neighbors, sn)
        assert np.array_equal(part.owned_local, owned)
        assert np.array_equal(part.local_to_global, verts)
        assert np.array_equal(part.subgraph.labels, g.labels[verts])


def test_cl5_deferred_big_rows(monkeypatch):
    # k = 5 rows with 128 < |R_i| <= 256 go to the CTA-wide compressed phase;
    # a dense RMAT has them (oriented hubs with d+ > 256)
    g = GR.from_edges_device(G.rmat_edges(16, 48, 2), num_vertices=1 << 16)
    og = pm.orient(g)
    assert og.max_degree > 256
    f = PL.as_forest(make_plan(P.generate_clique(5), g, oriented=True))
    tasks = EX._default_tasks(og, f)
    want = EX.execute(og, f, tasks, lgs=False)[0]
    for big in ("1", "0"):
        monkeypatch.setenv("G2M_CL5_BIG", big)
        og2 = pm.orient(g)
        assert EX.execute(og2, f, EX._default_tasks(og2, f))[0] == want, big


@pytest.mark.parametrize("core", ["0", "3", "9", "12", "16"])
@pytest.mark.parametrize("cta", ["0", "1"])
def test_hub_core_pair_tests(monkeypatch, core, cta):
    # pair-tier edge tests and CTA-tier rows through the hub-core bit matrix
    # (top 2^core ranks); a dense RMAT puts sources in every CTA tier
    g = GR.from_edges(G.rmat_edges(14, 40, 9), num_vertices=1 << 14)
    monkeypatch.setenv("G2M_PAIR_CORE", core)
    monkeypatch.setenv("G2M_CTA_CORE", cta)
    og = pm.orient(g)
    for k in (3, 4, 5):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        tasks = EX._default_tasks(og, f)
        assert EX.execute(og, f, tasks)[0] == EX.execute(og, f, tasks, lgs=False)[0], (core, k)


@pytest.mark.parametrize("rounds", ["0", "1"])
def test_cycle4_coarse_staging_rounds(monkeypatch, rounds):
    # the coarse staging tier (forced) with and without the batched count rounds
    g = GR.from_edges(G.rmat_edges(14, 16, 8), num_vertices=1 << 14)
    f = PL.as_forest(make_plan(cycle4(), g))
    want = EX.execute(g, f, EX._default_tasks(g, f), lgs=False)[0]
    monkeypatch.setenv("G2M_C4_FINE", "0")
    monkeypatch.setenv("G2M_C4_ROUNDS", rounds)
    g2 = GR.from_edges(G.rmat_edges(14, 16, 8), num_vertices=1 << 14)
    assert EX.execute(g2, f, EX._default_tasks(g2, f))[0] == want


def _rank_host(g, sym_deg):
    """Host restatement of the rank relabelling: rank = position in the
    (degree, id) order; row rank[v] = sorted rank[w], w in N(v)."""
    n = g.num_vertices
    off = np.asarray(g.row_offsets, dtype=np.int64)
    order = np.lexsort((np.arange(n), sym_deg))
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    deg = np.diff(off)
    roff = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg[order], out=roff[1:])
    rnbr = np.empty(int(off[-1]), dtype=np.int64)
    for v in range(n):
        r = rank[v]
        rnbr[roff[r]:roff[r + 1]] = np.sort(rank[g.neighbors[off[v]:off[v + 1]].astype(np.int64)])
    return roff, rnbr


def _row_class_graph():
    """Rows of every length class of the rank build (in-tile rows <= 32 slots,
    rows across 4096-slot tile edges, warp register sorts up to 256 / 512 /
    1024, CTA sorts beyond), runs of isolated vertices inside tiles, and a
    slot count that is not a multiple of 32."""
    n = 9000
    rng = np.random.default_rng(17)
    e = [np.column_stack([rng.integers(0, n, 30001), rng.integers(0, n, 30001)])]
    for hub, k in ((100, 33), (200, 200), (300, 300), (400, 700), (500, 1100), (600, 2500), (700, 31)):
        nb = rng.choice(np.arange(4000, n), size=k, replace=False)
        e.append(np.column_stack([np.full(k, hub), nb]))
    ed = np.concatenate(e)
    ed = ed[(ed[:, 0] != ed[:, 1]) & ((ed[:, 0] < 1500) | (ed[:, 0] >= 2500)) & ((ed[:, 1] < 1500) | (ed[:, 1] >= 2500))]
    return GR.from_edges(ed, num_vertices=n)     # ids 1500..2499 isolated


def test_rank_copy_equals_host_restatement():
    g = _row_class_graph()
    assert g.max_degree > 1024 and int(np.asarray(g.row_offsets)[-1]) % 32 != 0
    sym_deg = np.diff(np.asarray(g.row_offsets, dtype=np.int64))
    for gg in (g, pm.orient(g)):   # symmetric rows, then the oriented DAG (degrees of g)
        roff, rnbr = _rank_host(gg, sym_deg)
        rg = GR.rank_relabel(gg)
        assert np.array_equal(np.asarray(rg.row_offsets, dtype=np.int64), roff)
        assert np.array_equal(rg.neighbors.astype(np.int64), rnbr)


def test_device_orientation_tiles_equal_host():
    """The slot-tile orientation on graphs whose rows span many tiles, whose
    tiles hold long runs of empty rows, and whose slot count is a tile
    multiple or not."""
    for g in (_row_class_graph(), GR.from_edges(np.column_stack([np.zeros(5000, np.int64),
                                                                 np.arange(1, 5001)]), num_vertices=20000)):
        og = pm.orient(g)
        ho = orient_host(g)
        assert og == ho and og.oriented


def _support_share(g, rr, device=0):
    """One rank's support array (torch int32 on the device) and slot count."""
    import ctypes as C
    import torch
    from paper_2112_09761_b200 import _native as N
    dg = g.device_graph(device)
    n = C.c_uint64(0)
    N.check(N.lib().g2m_diamond_support(dg.handle, None, None, C.byref(n), None), "support")
    t = torch.zeros(max(int(n.value), 1), dtype=torch.int32, device=f"cuda:{device}")
    spec = EX.source_spec(rr, family="lgs")
    N.check(N.lib().g2m_diamond_support(dg.handle, C.byref(spec), C.c_void_p(t.data_ptr()), C.byref(n), None),
            "support")
    return t, int(n.value)


def _choose2(g, t, lo, hi, device=0):
    import ctypes as C
    from paper_2112_09761_b200 import _native as N
    w = np.zeros(2, dtype=np.uint64)
    N.check(N.lib().g2m_support_choose2(g.device_graph(device).handle, C.c_void_p(t.data_ptr()), lo, hi,
                                        N.ptr(w, C.c_uint64), None), "choose2")
    return int(w[0]) | (int(w[1]) << 64)


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_diamond_support_split_allreduce_equals_single(parts):
    """The multi-GPU diamond path with the all-reduce done by hand: the
    ranks' support arrays (source shares, estimator split) summed, then
    C(t, 2) over each rank's slot share, add up to the one-device count and
    to the oracle; and the summed array equals the unsplit support."""
    import torch
    from util import diamond
    g = GR.from_edges(G.rmat_edges(12, 8, 21), num_vertices=1 << 12)
    want = pm.subgraph_listing(g, diamond(), mode="count").counts["diamond"]
    full, n = _support_share(g, None)
    acc = torch.zeros_like(full)
    for i in range(parts):
        t, _ = _support_share(g, (256, parts, i) if parts > 1 else None)
        acc += t
    torch.cuda.synchronize()
    assert torch.equal(acc, full)
    got = sum(_choose2(g, acc, i * n // parts, (i + 1) * n // parts) for i in range(parts))
    assert got == want
    f, gg = forest_for_diamond(g)
    assert want == O.run(gg, f, threads=4)[0]["diamond"]


def forest_for_diamond(g):
    from test_oracle import forest_for
    return forest_for("diamond", g)


def test_bench_multi_rank_diamond_allreduce_gloo():
    # two ranks folded onto one GPU (gloo): support shares, one all-reduce of
    # the support array, C(t, 2) per slot share; counts equal the one-rank run
    common = ["--workload", "diamond", "--scale", "14", "--steps", "2", "--warmup", "1",
              "--no-cpu-baseline", "--no-e2e", "--no-roofline", "--no-parity"]
    one = _bench(common)
    two = _bench(common + ["--gpus", "2"], {"G2M_BENCH_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["counts"] == two["counts"]
    assert "all-reduce of the per-edge support array" in two["config"]["parallelism"]
