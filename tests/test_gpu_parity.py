"""GPU parity: the generated sm_100a kernels, called through the public API
and the C ABI, give the reference's exact counts (golden fixtures), the
oracle's exact counts on larger seeded graphs, and the reference's exact list
streams."""
import json
from math import comb
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
from paper_2112_09761_b200 import scheduler, setops
from test_oracle import COUNTS, LISTS, build_graph, forest_for
from util import analyze, complete, cycle4, diamond, er, make_plan, orient_host

pytestmark = pytest.mark.gpu


def api_counts(g, w):
    if w == "tc":
        return {"triangle": pm.triangle_count(g)}
    if w in ("4-clique", "5-clique"):
        return pm.k_clique(g, int(w[0])).counts
    if w == "4-cycle":
        return pm.subgraph_listing(g, cycle4(), mode="count").counts
    if w == "diamond":
        return pm.subgraph_listing(g, diamond(), mode="count").counts
    return {p.name: c for p, c in pm.k_motif(g, int(w[0])).items()}


_gc = {}


def gg(key):
    if key not in _gc:
        _gc[key] = build_graph(key, COUNTS[key])
    return _gc[key]


CASES = [(k, w) for k in sorted(COUNTS) for w in sorted(COUNTS[k]["counts"])]


@pytest.mark.parametrize("key,workload", CASES)
def test_api_counts_match_reference_golden(key, workload):
    assert api_counts(gg(key), workload) == COUNTS[key]["counts"][workload]


@pytest.mark.parametrize("flatten", [True, False])
@pytest.mark.parametrize("workload", ["tc", "4-clique", "5-clique", "4-cycle", "diamond", "3-motif", "4-motif"])
def test_kernel_variants_match_oracle_rmat(workload, flatten):
    scale = 9 if workload == "4-motif" else 12
    g = GR.from_edges(G.rmat_edges(scale, 16, 5), num_vertices=1 << scale)
    forest, gh = forest_for(workload, g)
    want, _ = O.run(gh, forest)
    gd = GR.orient(g) if gh.oriented else g
    got, _, _, _ = EX.execute(gd, forest, EX._default_tasks(gd, forest), flatten=flatten)
    assert got == want


def test_powerlaw_three_motif_matches_oracle():
    g = GR.from_edges(G.powerlaw_edges(20000, 4, 3), num_vertices=20000)
    res = {p.name: c for p, c in pm.k_motif(g, 3).items()}
    assert res == {"wedge": 2037726, "triangle": 1598}   # reference


def test_rmat12_known_counts():
    g = GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12)
    assert g.num_edges // 2 == 48222
    assert pm.triangle_count(g) == 480521
    assert pm.k_clique(g, 4).counts["4-clique"] == 4056943
    assert pm.k_clique(g, 5).counts["5-clique"] == 27268396
    assert pm.subgraph_listing(g, diamond(), mode="count").counts["diamond"] == 57343012
    assert pm.subgraph_listing(g, cycle4(), mode="count").counts["4-cycle"] == 52799071


def _hub_graph(scale=12):
    """R-MAT plus rows longer than the warp row passes take (g2m.cu kHubRow =
    2048, kRowSortWarp = 1024; at scale 14 also > kRowSortBlock = 8192)."""
    n = 1 << scale
    e = [G.rmat_edges(scale, 8, 5)]
    for hub, k in ((7, n - 1), (9, 3000), (4000, 2049), (11, 2048), (13, 1025), (15, 1024), (17, 33)):
        others = np.array([v for v in range(k + 1) if v != hub][:k], dtype=np.int64)
        e.append(np.column_stack([np.full(len(others), hub), others]))
    return GR.from_edges(np.concatenate(e), num_vertices=n)


def test_device_orientation_equals_host():
    for g in (GR.from_edges(G.rmat_edges(11, 16, 3), num_vertices=1 << 11), _hub_graph()):
        og = GR.orient(g)
        ho = orient_host(g)
        assert og == ho and og.max_degree == ho.max_degree and og.oriented


def test_hub_rows_rank_build():
    """Hub rows go through the block-per-row passes of orientation and the
    rank relabelling; the rank-space kernels must still equal the generated
    kernels on the original ids."""
    g = _hub_graph()
    assert g.max_degree > 4000
    for gs in (g, _hub_graph(14)):
        for pat, rw in ((cycle4(), False), (diamond(), True)):
            f = PL.as_forest(make_plan(pat, gs, rewrite=rw))
            tasks = EX._default_tasks(gs, f)
            assert EX.execute(gs, f, tasks, lgs=True)[0] == EX.execute(gs, f, tasks, lgs=False)[0]
    og = orient_host(g)
    want = {}
    for k in (3, 4):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        tasks = EX._default_tasks(og, f)
        want[k] = EX.execute(og, f, tasks, lgs=False)[0]
        assert EX.execute(og, f, tasks, lgs=True)[0] == want[k]
    # public API: device orientation (hub blocks) -> rank build -> LGS
    assert pm.triangle_count(g) == want[3]["triangle"]
    assert pm.k_clique(g, 4).counts == want[4]


def test_rank_build_many_block_rows():
    """K_1100: every row (1,099 slots) takes the block row sort, more rows than
    slots / 2048 (hub-list capacity per row threshold)."""
    g = complete(1100)
    assert pm.subgraph_listing(g, cycle4(), mode="count").counts["4-cycle"] == 3 * comb(1100, 4)
    assert pm.triangle_count(g) == comb(1100, 3)


def test_rank_row_sort_equals_radix(monkeypatch):
    """The per-row rank-space build and the global key sort give the same counts."""
    g = _hub_graph(12)   # rows up to 4095: warp and block row sorts
    f = PL.as_forest(make_plan(cycle4(), g))
    tasks = EX._default_tasks(g, f)
    a = EX.execute(g, f, tasks)[0]
    g2 = _hub_graph(12)
    monkeypatch.setenv("G2M_RANK_RADIX", "1")
    assert EX.execute(g2, f, tasks)[0] == a


def test_device_csr_builder_equals_host():
    e = G.rmat_edges(12, 8, 4)
    a = GR.from_edges(e, num_vertices=1 << 12)
    b = GR.from_edges_device(e, num_vertices=1 << 12)
    assert a == b and a.max_degree == b.max_degree


def test_explicit_and_shuffled_tasks():
    g = er(45, 0.25, 12)
    pl = make_plan(diamond(), g)
    tasks = pm.build_edge_tasks(g, pl)
    base = pm.run_dfs(g, pl, tasks=tasks).counts
    explicit = GR.EdgeTaskList(tasks.edges.copy(), reduced=True)
    assert pm.run_dfs(g, pl, tasks=explicit).counts == base
    rng = np.random.default_rng(0)
    for _ in range(5):
        perm = rng.permutation(len(tasks.edges))
        shuffled = GR.EdgeTaskList(tasks.edges[perm], reduced=True)
        assert pm.run_dfs(g, pl, tasks=shuffled).counts == base
    full = GR.EdgeTaskList(GR.all_edge_tasks(g), reduced=False)
    assert pm.run_dfs(g, pl, tasks=full).counts == base


def test_vertex_and_edge_parallel_agree():
    g = er(40, 0.25, 3)
    for p in [diamond(), cycle4(), P.generate_clique(3)] + P.generate_all_motifs(4):
        ce = pm.run_dfs(g, make_plan(p, g, granularity="edge")).counts
        cv = pm.run_dfs(g, make_plan(p, g, granularity="vertex")).counts
        assert ce == cv, p.name


def test_random_patterns_vs_oracle():
    rng = np.random.default_rng(2024)
    cases = 0
    while cases < 25:
        k = int(rng.integers(3, 6))
        pairs = [(a, b) for a in range(k) for b in range(a + 1, k)]
        keep = [e for e in pairs if rng.random() < 0.55]
        induced = "vertex" if rng.random() < 0.5 else "edge"
        try:
            p = P.Pattern(k, keep, induced=induced)
        except ValueError:
            continue
        cases += 1
        g = er(26 if k == 5 else 34, 0.25, int(rng.integers(1 << 30)))
        gran = "vertex" if rng.random() < 0.5 else "edge"
        pl = make_plan(p, g, granularity=gran)
        want, _ = O.run(g, PL.as_forest(pl))
        assert pm.run_dfs(g, pl).counts == want, (k, keep, induced, gran)


def test_labeled_patterns_vs_oracle():
    g = er(40, 0.25, 16, labels=3)
    for edges, labels in ([((0, 1),), (0, 1)], [((0, 1), (0, 2)), (2, 0, 1)],
                          [((0, 1), (0, 2), (1, 2)), (1, 1, 2)]):
        p = P.Pattern(len(labels), edges, labels=labels)
        for gran in ("edge", "vertex"):
            pl = make_plan(p, g, granularity=gran)
            want, _ = O.run(g, PL.as_forest(pl))
            assert pm.run_dfs(g, pl).counts == want, (labels, gran)


@pytest.mark.parametrize("key", sorted(LISTS))
def test_list_stream_exact_reference_order(key):
    gk, pk, gran = key.split("|")
    _, n, p, s = gk.split("/")
    g = er(int(n), float(p), int(s))
    pats = {"triangle": P.generate_clique(3), "4-clique": P.generate_clique(4),
            "diamond": diamond(), "4-cycle": cycle4(),
            "tailed": P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2)], induced="vertex")}
    pat = pats[pk]
    mo, so = analyze(pat, g)
    pl = PL.build_plan(pat, mo, so, "list", granularity=gran)
    stream = []
    res = pm.run_dfs(g, pl, sink=lambda pid, m: (stream.append(m), False)[1])
    assert stream == [tuple(m) for m in LISTS[key]["stream"]]
    assert res.counts[pat.name] == len(stream) and not res.stopped_early


def test_early_termination():
    g = er(30, 0.3, 8)
    res = pm.run_dfs(g, make_plan(diamond(), g, mode="list"), sink=lambda pid, m: True)
    assert res.stopped_early and sum(res.counts.values()) == 1
    seen = []
    res = pm.run_dfs(g, make_plan(cycle4(), g, mode="list"),
                     sink=lambda pid, m: (seen.append(m), len(seen) >= 7)[1])
    assert res.stopped_early and res.counts["4-cycle"] == 7 == len(seen)


def test_list_mode_without_sink_counts():
    g = er(50, 0.2, 5)
    for p in (diamond(), cycle4(), P.generate_clique(4)):
        a = pm.run_dfs(g, make_plan(p, g, mode="list")).counts
        b = pm.run_dfs(g, make_plan(p, g, mode="count")).counts
        assert a == b


def test_apps_surface():
    assert pm.triangle_count(complete(4)) == 4
    assert pm.triangle_count(pm.from_edges([(i, (i + 1) % 5) for i in range(5)])) == 0
    assert pm.k_clique(complete(6), 5).counts["5-clique"] == 6
    for k in (6, 7, 8):
        assert pm.k_clique(complete(9), k).counts[f"{k}-clique"] == comb(9, k)
    assert pm.subgraph_listing(complete(4), cycle4(), mode="count").counts["4-cycle"] == 3
    assert pm.subgraph_listing(complete(4), diamond(), mode="count").counts["diamond"] == 6
    assert {p.name: c for p, c in pm.k_motif(complete(4), 3).items()} == {"wedge": 0, "triangle": 4}
    res = pm.run_job(pm.MiningJob(graph=complete(4), patterns=[P.generate_clique(3)]))
    assert res.applied("orientation")
    og = pm.orient(complete(4))
    assert pm.run_job(pm.MiningJob(graph=og, patterns=[P.generate_clique(3)])).counts["triangle"] == 4
    g = er(60, 0.2, 3)
    on = pm.k_clique(g, 4, cfg=pm.ExecutionConfig(lgs="auto", lgs_delta_threshold=10 ** 6))
    off = pm.k_clique(g, 4, cfg=pm.ExecutionConfig(lgs="auto", lgs_delta_threshold=1))
    assert on.applied("local-graph-search") and not off.applied("local-graph-search")
    assert on.counts == off.counts
    seen = []
    g = er(60, 0.15, 7)
    cnt = pm.subgraph_listing(g, diamond(), mode="count").counts["diamond"]
    pm.subgraph_listing(g, diamond(), mode="list", sink=lambda pid, m: (seen.append(m), False)[1])
    assert len(seen) == cnt


def test_errors_match_reference():
    og = pm.orient(complete(4))
    with pytest.raises(ValueError, match="orientation"):
        pm.run_dfs(og, make_plan(P.generate_clique(3)))
    with pytest.raises(ValueError, match="orientation"):
        pm.run_dfs(complete(4), make_plan(P.generate_clique(3), oriented=True))
    with pytest.raises(ValueError):
        pm.run_dfs(complete(4), make_plan(diamond(), granularity="vertex"),
                   tasks=pm.build_edge_tasks(complete(4), make_plan(diamond())))
    with pytest.raises(ValueError, match="hub"):
        pm.run_dfs_lgs(complete(4), make_plan(cycle4()))
    with pytest.raises(ValueError, match="vertex granularity"):
        pm.run_dfs_lgs(complete(4), make_plan(P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2)])))
    with pytest.raises(pm.BudgetError):
        pm.run_dfs(er(20, 0.3, 1), make_plan(P.generate_clique(4), mode="list"),
                   cfg=pm.ExecutionConfig(memory_budget=1))


def test_lgs_entry_matches_dfs():
    g = er(200, 0.08, 21)
    og = pm.orient(g)
    for k in (4, 5):
        pl = make_plan(P.generate_clique(k), g, oriented=True)
        assert pm.run_dfs_lgs(og, pl).counts == pm.run_dfs(og, pl).counts
    g = er(60, 0.25, 2)
    for mode in ("count", "list"):
        pl = make_plan(diamond(), g, mode=mode)
        assert pm.run_dfs_lgs(g, pl).counts == pm.run_dfs(g, pl).counts


def test_budgeted_worker_formula():
    g = er(60, 0.2, 5)
    pl = make_plan(P.generate_clique(4), g, mode="list")
    tasks = pm.build_edge_tasks(g, pl)
    for budget in (g.max_degree * 4, g.max_degree * 4 * 5, g.max_degree * 4 * 10 ** 6):
        res = pm.run_dfs(g, pl, tasks=tasks, cfg=pm.ExecutionConfig(memory_budget=budget))
        want = min(budget // (pl.num_buffers * g.max_degree * 4), len(tasks))
        assert res.stats.workers == max(1, want)
        assert all(h <= g.max_degree for h in res.stats.buffer_high_water)


def test_scheduler_invariance_and_reports():
    g = er(64, 0.2, 77)
    pl = make_plan(diamond(), g)
    tasks = pm.build_edge_tasks(g, pl)
    base = pm.run_dfs(g, pl, tasks=tasks).counts
    for n in (1, 2, 4, 8):
        for policy in (scheduler.POLICY_EVEN, scheduler.POLICY_RR, scheduler.POLICY_CHUNKED):
            sched = scheduler.make_schedule(tasks, n, policy, workers_y=2)
            res = scheduler.run_on_devices(g, pl, sched, tasks, parallel=False)
            assert res.counts == base, (n, policy)
            assert len(res.reports) == n
    sched = scheduler.split_even(tasks, 1)
    res = scheduler.run_on_devices(g, pl, sched, tasks, parallel=False)
    assert res.load_report_csv().splitlines()[0] == "device_id,tasks,elapsed_ms,count"
    single = pm.run_job(pm.MiningJob(graph=g, patterns=[diamond()]))
    multi = pm.run_job(pm.MiningJob(graph=g, patterns=[diamond()], devices=2,
                                    parallel_devices=False))
    assert multi.counts == single.counts and len(multi.devices.reports) == 2


def test_hub_partition():
    pl = make_plan(P.generate_clique(5), granularity="vertex")
    res = scheduler.run_partitioned_hub(complete(6), pl, 2)
    assert res.counts == {"5-clique": 6}
    g = er(300, 0.05, 9)
    pl = make_plan(P.generate_clique(4), g, granularity="vertex")
    whole = pm.run_dfs(g, pl, tasks=np.arange(g.num_vertices)).counts
    for n in (2, 4):
        assert scheduler.run_partitioned_hub(g, pl, n).counts == whole


def test_setops_fuzz_against_merge_scan():
    rng = np.random.default_rng(4242)
    A, B, BD = [], [], []
    for _ in range(3000):
        A.append(np.unique(rng.integers(0, 200, int(rng.integers(0, 60))).astype(np.uint32)))
        B.append(np.unique(rng.integers(0, 200, int(rng.integers(0, 60))).astype(np.uint32)))
        BD.append(int(rng.integers(0, 220)) if rng.random() < 0.5 else None)
    ci, li = setops.setop_batch(setops.OP_INTERSECT, A, B, BD)
    cc, _ = setops.setop_batch(setops.OP_INTERSECT_COUNT, A, B, BD)
    di, ld = setops.setop_batch(setops.OP_DIFFERENCE, A, B, BD)
    dc, _ = setops.setop_batch(setops.OP_DIFFERENCE_COUNT, A, B, BD)
    for i in range(len(A)):
        bs = set(B[i].tolist())
        inter = [x for x in A[i].tolist() if x in bs and (BD[i] is None or x < BD[i])]
        diff = [x for x in A[i].tolist() if x not in bs and (BD[i] is None or x < BD[i])]
        assert li[i].tolist() == inter and cc[i] == len(inter) == ci[i]
        assert ld[i].tolist() == diff and dc[i] == len(diff) == di[i]
    assert setops.intersect(np.array([1, 3, 5], np.uint32), np.array([3, 4, 5], np.uint32)).tolist() == [3, 5]
    assert setops.intersect_count(np.array([1, 3, 5], np.uint32), np.array([3, 4, 5], np.uint32), bound=5) == 1


def test_empty_graphs():
    g = pm.from_edges(np.empty((0, 2), dtype=np.int64), num_vertices=0)
    assert pm.run_dfs(g, make_plan(diamond())).counts["diamond"] == 0
    gv = pm.from_edges(np.empty((0, 2), dtype=np.int64), num_vertices=5)
    assert pm.run_dfs(gv, make_plan(P.generate_clique(3))).counts["triangle"] == 0
    assert pm.triangle_count(gv) == 0


BALG = json.loads((Path(__file__).parent / "golden" / "balg.json").read_text())


@pytest.mark.parametrize("key", sorted(BALG))
def test_instrumented_kernel_bytes_match_reference(key):
    """The instrumented generated kernel reproduces the SURVEY 8(d)
    algorithmic bytes of the instrumented reference exactly."""
    if key.startswith("er/"):
        _, n, p, s = key.split("/")
        g = er(int(n), float(p), int(s))
    else:
        g = GR.from_edges(G.rmat_edges(10, 16, 1), num_vertices=1 << 10)
    for w, want in BALG[key].items():
        forest, gh = forest_for(w, g)
        gd = GR.orient(g) if gh.oriented else g
        assert EX.algorithmic_bytes(gd, forest) == want, (key, w)


@pytest.mark.parametrize("workload", ["4-motif", "4-clique", "4-cycle"])
def test_instrumented_bytes_match_oracle_rmat11(workload):
    g = GR.from_edges(G.rmat_edges(11 if workload != "4-motif" else 9, 16, 2),
                      num_vertices=1 << (11 if workload != "4-motif" else 9))
    forest, gh = forest_for(workload, g)
    _, want = O.run(gh, forest)
    gd = GR.orient(g) if gh.oriented else g
    assert EX.algorithmic_bytes(gd, forest) == want


def _heavy_source_graph(na=1100, p=0.02):
    """A source u with out-degree na (1100: the W=32/64 tiers; 2100: beyond
    them, the generic fallback for k > 3): u links to A (na vertices); each a
    in A gets na+1 private leaves so deg(a) > deg(u); A is internally an ER
    graph so cliques through u exist."""
    rng = np.random.default_rng(11)
    leaves = na + 1
    A = np.arange(1, na + 1)
    edges = [np.column_stack([np.zeros(na, dtype=np.int64), A])]
    mask = np.triu(rng.random((na, na)) < p, 1)
    ii, jj = np.nonzero(mask)
    edges.append(np.column_stack([A[ii], A[jj]]))
    base = na + 1
    src = np.repeat(A, leaves)
    dst = base + np.arange(na * leaves)
    edges.append(np.column_stack([src, dst]))
    e = np.concatenate(edges).astype(np.int64)
    return GR.from_edges(e, num_vertices=base + na * leaves)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_lgs_clique_kernels_match_generic_and_oracle(k):
    graphs = [complete(9), complete(70), er(200, 0.08, 21), er(150, 0.3, 5),
              GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12),
              GR.from_edges(G.rmat_edges(14, 16, 3), num_vertices=1 << 14),
              _heavy_source_graph(), _heavy_source_graph(2100)]
    for g in graphs:
        og = GR.orient(g)
        pl = make_plan(P.generate_clique(k), g, oriented=True)
        f = PL.as_forest(pl)
        tasks = EX._default_tasks(og, f)
        a, _, _, _ = EX.execute(og, f, tasks, lgs=True)
        b, _, _, _ = EX.execute(og, f, tasks, lgs=False)
        assert a == b, (g, k)
        if g.num_edges < 300000:
            want, _ = O.run(orient_host(g), f)
            assert a == want
    assert pm.k_clique(complete(70), 5).counts["5-clique"] == comb(70, 5)
    assert pm.k_clique(complete(64), 4).counts["4-clique"] == comb(64, 4)
    assert pm.k_clique(complete(65), 4).counts["4-clique"] == comb(65, 4)
    big = complete(1200)      # out-degrees 0..1199: every tier incl. W=32/64
    for kk in (3, 4, 5):
        assert list(pm.k_clique(big, kk).counts.values()) == [comb(1200, kk)]


@pytest.mark.parametrize("k", [4, 5])
def test_lgs_global_slab_tier_medium_density(k):
    """A source with out-degree 1100 (the global-slab W = 32 tier) whose local
    graph is ER p = 0.3: rows of ~330 members, k = 5 pairs both light and
    heavy (> 32 common members); bitmap LGS = plan kernel."""
    g = _heavy_source_graph(1100, 0.3)
    og = GR.orient(g)
    f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
    tasks = EX._default_tasks(og, f)
    a, _, _, _ = EX.execute(og, f, tasks, lgs=True)
    b, _, _, _ = EX.execute(og, f, tasks, lgs=False)
    assert a == b


def test_rmat12_lgs_known_counts():
    g = GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12)
    for k, want in ((3, 480521), (4, 4056943), (5, 27268396)):
        og = GR.orient(g)
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        got, _, _, _ = EX.execute(og, f, EX._default_tasks(og, f), lgs=True)
        assert got[f.pattern_ids[0]] == want


def test_cycle4_wedge_kernels_match_generic_and_oracle():
    """g2m_cycle4_count (warp / CTA-hash / dense-HBM tiers) == the generated
    4-cycle plan kernel == the oracle; K_n has 3*C(n,4) 4-cycles."""
    graphs = [complete(4), complete(30), er(200, 0.1, 17), er(120, 0.3, 4),
              GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12),
              GR.from_edges(G.rmat_edges(14, 16, 2), num_vertices=1 << 14),
              GR.from_edges(G.powerlaw_edges(5000, 4, 3), num_vertices=5000)]
    for g in graphs:
        pl = make_plan(cycle4(), g)
        f = PL.as_forest(pl)
        tasks = EX._default_tasks(g, f)
        a, _, _, _ = EX.execute(g, f, tasks, lgs=True)
        b, _, _, _ = EX.execute(g, f, tasks, lgs=False)
        assert a == b, g
        if g.num_edges < 100000:
            want, _ = O.run(g, f)
            assert a == want
    assert pm.subgraph_listing(complete(30), cycle4(), mode="count").counts["4-cycle"] == 3 * comb(30, 4)
    g = GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12)
    assert pm.subgraph_listing(g, cycle4(), mode="count").counts["4-cycle"] == 52799071
    # chunked round-robin shares of the top vertex add up to the whole
    f = PL.as_forest(make_plan(cycle4(), g))
    tasks = EX._default_tasks(g, f)
    parts = [EX.execute(g, f, tasks, rr=(64, 3, i))[0]["4-cycle"] for i in range(3)]
    assert sum(parts) == 52799071


def test_cycle4_grid_tier(monkeypatch):
    """A small staging cap sends the large wedge fans to the grid-wide tier."""
    g = GR.from_edges(G.rmat_edges(13, 16, 4), num_vertices=1 << 13)
    f = PL.as_forest(make_plan(cycle4(), g))
    tasks = EX._default_tasks(g, f)
    want = EX.execute(g, f, tasks, lgs=False)[0]
    monkeypatch.setenv("G2M_C4_STAGE_CAP", "20000")
    assert EX.execute(g, f, tasks)[0] == want


@pytest.mark.parametrize("fine", ["0", "1"])
def test_cycle4_stage_bucket_variants(monkeypatch, fine):
    """Staged tier with 32K-id coarse buckets (k_c4_stage2) and 1024-id fine
    buckets (k_c4_stage), with a stage cap that also sends v1s to the grid tier."""
    g = GR.from_edges(G.rmat_edges(16, 8, 6), num_vertices=1 << 16)   # r1 > 32K: several coarse buckets
    f = PL.as_forest(make_plan(cycle4(), g))
    tasks = EX._default_tasks(g, f)
    want = EX.execute(g, f, tasks, lgs=False)[0]
    monkeypatch.setenv("G2M_C4_FINE", fine)
    assert EX.execute(g, f, tasks)[0] == want
    monkeypatch.setenv("G2M_C4_STAGE_CAP", "100000")
    assert EX.execute(g, f, tasks)[0] == want


def test_diamond_support_kernels_match_generic_and_oracle():
    """g2m_diamond_count (edge triangle support over the rank-space DAG) ==
    the generated diamond plan kernel (counting rewrite) == the oracle."""
    graphs = [complete(4), complete(40), er(200, 0.1, 17), er(120, 0.3, 4),
              GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12),
              GR.from_edges(G.rmat_edges(14, 16, 2), num_vertices=1 << 14),
              GR.from_edges(G.powerlaw_edges(5000, 4, 3), num_vertices=5000),
              _heavy_source_graph()]
    for g in graphs:
        pl = make_plan(diamond(), g, rewrite=True)
        f = PL.as_forest(pl)
        tasks = EX._default_tasks(g, f)
        a, _, _, _ = EX.execute(g, f, tasks, lgs=True)
        b, _, _, _ = EX.execute(g, f, tasks, lgs=False)
        assert a == b, g
        if g.num_edges < 100000:
            want, _ = O.run(g, f)
            assert a == want
    assert pm.subgraph_listing(complete(40), diamond(), mode="count").counts["diamond"] == 6 * comb(40, 4)
    g = GR.from_edges(G.rmat_edges(12, 16, 1), num_vertices=1 << 12)
    assert pm.subgraph_listing(g, diamond(), mode="count").counts["diamond"] == 57343012


@pytest.mark.parametrize("chunk,fbytes", [(1, None), (7, None), (32, None), (32, 4096)])
def test_bounded_bfs_equals_dfs(chunk, fbytes):
    """The bounded-frontier BFS runtime (expand/consume kernels, blocks
    redone on frontier overflow) gives the DFS counts for every forest with
    a level-3 subtree: 4-motifs (fused), 4-cycle, diamond list plan,
    5-cycle; explicit shuffled tasks too (reference BFS/DFS agreement,
    test_executor.py:228-235)."""
    graphs = [er(60, 0.2, 3), GR.from_edges(G.powerlaw_edges(3000, 4, 3), num_vertices=3000),
              GR.from_edges(G.rmat_edges(10, 8, 2), num_vertices=1 << 10)]
    forests = [PL.fuse_multi_pattern([make_plan(p, rewrite=True) for p in P.generate_all_motifs(4)]),
               PL.as_forest(make_plan(cycle4())),
               PL.as_forest(make_plan(diamond(), mode="list")),
               PL.as_forest(make_plan(P.Pattern(5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)])))]
    cfg = EX.ExecutionConfig(search="bfs", bfs_chunk=chunk, frontier_bytes=fbytes)
    for g in graphs:
        for f in forests:
            tasks = EX._default_tasks(g, f)
            want, _, _, _ = EX.execute(g, f, tasks, lgs=False)
            got, st, _, _ = EX.execute(g, f, tasks, lgs=False, search="bfs", cfg=cfg)
            assert got == want, (g, f.pattern_ids)
            if fbytes:
                assert st.high_water[6] > 1       # ran in several bounded blocks
    g = graphs[1]
    f = forests[0]
    tasks = GR.EdgeTaskList(GR.all_edge_tasks(g), reduced=False)
    perm = np.random.default_rng(1).permutation(len(tasks.edges))
    shuffled = GR.EdgeTaskList(tasks.edges[perm], reduced=False)
    want = EX.execute(g, f, shuffled, lgs=False)[0]
    assert EX.execute(g, f, shuffled, lgs=False, search="bfs", cfg=cfg)[0] == want


def test_kmotif_bfs_log_and_counts():
    g = GR.from_edges(G.powerlaw_edges(20000, 4, 3), num_vertices=20000)
    res = pm.run_job(pm.MiningJob(graph=g, patterns=P.generate_all_motifs(4), granularity="edge"))
    assert res.applied("bounded-bfs")
    dfs = pm.run_job(pm.MiningJob(graph=g, patterns=P.generate_all_motifs(4), granularity="edge",
                                  cfg=EX.ExecutionConfig(search="dfs")))
    assert not dfs.applied("bounded-bfs")
    assert res.counts == dfs.counts


def _rmat_device_host_restatement(scale, ef, seed, a=0.57, b=0.19, c=0.19):
    """numpy restatement of k_rmat_keys (g2m.cu): splitmix-style hash of
    (seed, edge, bit) -> uniform double -> quadrant bits."""
    m = ef << scale
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    i = np.arange(m, dtype=np.uint64)
    u = np.zeros(m, dtype=np.uint64)
    v = np.zeros(m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for bit in range(scale):
            z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + i * np.uint64(0xD1B54A32D192ED03)
                 + np.uint64(bit) * np.uint64(0xABC98388FB8FAC03)) & M
            z ^= z >> np.uint64(30); z = (z * np.uint64(0xBF58476D1CE4E5B9)) & M
            z ^= z >> np.uint64(27); z = (z * np.uint64(0x94D049BB133111EB)) & M
            z ^= z >> np.uint64(31)
            r = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
            u |= (r >= a + b).astype(np.uint64) << np.uint64(bit)
            v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.uint64) << np.uint64(bit)
    return np.column_stack([u.astype(np.int64), v.astype(np.int64)])


def test_device_rmat_generator_equals_host_restatement():
    g = GR.rmat_device(11, 8, 3)
    h = GR.from_edges(_rmat_device_host_restatement(11, 8, 3), num_vertices=1 << 11)
    assert g == h and g.max_degree == h.max_degree
    want = pm.triangle_count(h)
    assert pm.triangle_count(g) == want


@pytest.mark.parametrize("direct_max", ["0", "4096"])
def test_lgs_two_level_window_matches(monkeypatch, direct_max):
    """Windows too wide for the direct bitmap use the two-level window (or the
    hash map): forced here by capping the direct bitmap."""
    g = GR.from_edges(G.rmat_edges(14, 16, 3), num_vertices=1 << 14)
    og = GR.orient(g)
    want = {}
    for k in (3, 4, 5):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        want[k] = EX.execute(og, f, EX._default_tasks(og, f), lgs=False)[0]
    monkeypatch.setenv("G2M_DIRECT_MAX", direct_max)
    for k in (3, 4, 5):
        f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
        assert EX.execute(og, f, EX._default_tasks(og, f))[0] == want[k], k
    # the diamond support path shares the CTA kernels
    pl = make_plan(diamond(), g, rewrite=True)
    fd = PL.as_forest(pl)
    td = EX._default_tasks(g, fd)
    monkeypatch.delenv("G2M_DIRECT_MAX")
    wd = EX.execute(g, fd, td, lgs=False)[0]
    monkeypatch.setenv("G2M_DIRECT_MAX", direct_max)
    assert EX.execute(g, fd, td)[0] == wd
