"""GPU parity of the generated bitmap local-graph-search kernels
(codegen_lgs) for hub-rooted plans -- counts and list streams against the
CPU oracle (the reference executor's restatement) and the sorted-list plan
kernel; the reference's LGS equals run_dfs exactly (executor.py:526-533)."""
import numpy as np
import pytest

import graphs as G
import paper_2112_09761_b200 as pm
from oracle import oracle as O
from paper_2112_09761_b200 import executor as EX
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import plan as PL
from util import TAILED_EDGES, diamond, er, make_plan

pytestmark = pytest.mark.gpu

BOOK = P.Pattern(5, [(0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (0, 4), (1, 4)])
STAR3 = P.Pattern(4, [(0, 1), (0, 2), (0, 3)])
WEDGE = P.Pattern(3, [(0, 1), (0, 2)])
TAILED = P.Pattern(4, TAILED_EDGES)
DIAMOND_V = P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)], induced="vertex")


def _graphs():
    yield "er80", er(80, 0.15, 3)
    yield "rmat9", GR.from_edges(G.rmat_edges(9, 8, 2), num_vertices=1 << 9)   # max degree > 64
    yield "pl3000", GR.from_edges(G.powerlaw_edges(3000, 4, 3), num_vertices=3000)  # > 256: global rows


CASES = [("diamond", diamond(), "edge"), ("diamond", diamond(), "vertex"),
         ("diamond-vi", DIAMOND_V, "edge"), ("book", BOOK, "edge"), ("tailed", TAILED, "vertex"),
         ("3-star", STAR3, "vertex"), ("wedge", WEDGE, "vertex")]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[2]}" for c in CASES])
@pytest.mark.parametrize("mode", ["count", "list"])
def test_lgs_counts_match_oracle(case, mode):
    name, pat, gran = case
    for gname, g in _graphs():
        if gname == "pl3000" and name in ("book", "3-star") and mode == "list":
            continue      # match streams of millions: the count pass covers them
        pl = make_plan(pat, g, mode=mode, granularity=gran)
        want, _ = O.run(g, PL.as_forest(pl), threads=8)
        got = pm.run_dfs_lgs(g, pl)
        assert got.counts == want, (gname, got.counts, want)
        if mode == "count":
            rw = make_plan(pat, g, granularity=gran, rewrite=True)
            assert pm.run_dfs_lgs(g, rw).counts == want, gname


@pytest.mark.parametrize("case", CASES[:5], ids=[f"{c[0]}-{c[2]}" for c in CASES[:5]])
def test_lgs_list_stream_in_reference_order(case):
    name, pat, gran = case
    for gname, g in list(_graphs())[:2]:
        pl = make_plan(pat, g, mode="list", granularity=gran)
        cap = 2_000_000
        want, _, stream = O.run(g, PL.as_forest(pl), threads=1, list_cap=cap)
        got = []
        res = pm.run_dfs_lgs(g, pl, sink=lambda pid, m: (got.append((pid, m)), False)[1])
        assert len(got) == sum(want.values()) and res.counts == want and not res.stopped_early
        assert got[:cap] == stream, gname      # the oracle keeps the first `cap` matches


def test_lgs_early_termination():
    g = er(40, 0.3, 8)
    seen = []
    res = pm.run_dfs_lgs(g, make_plan(diamond(), g, mode="list"),
                         sink=lambda pid, m: (seen.append(m), len(seen) >= 5)[1])
    assert res.stopped_early and len(seen) == 5


@pytest.mark.parametrize("k", [3, 4, 5, 6, 7])
@pytest.mark.parametrize("gran", ["edge", "vertex"])
def test_generated_lgs_cliques(monkeypatch, k, gran):
    # cliques k >= 6 always take the generated kernel; k <= 5 forced onto it
    monkeypatch.setattr(EX, "LGS_GENERATED_CLIQUES", True)
    g = GR.from_edges(G.rmat_edges(9, 16, 3), num_vertices=1 << 9)
    og = pm.orient(g)
    pl = make_plan(P.generate_clique(k), g, granularity=gran, oriented=True)
    want, _ = O.run(og, PL.as_forest(pl), threads=8)
    assert pm.run_dfs_lgs(og, pl).counts == want


def test_run_job_uses_generated_lgs_for_hub_patterns():
    g = er(120, 0.1, 4)
    job = pm.run_job(pm.MiningJob(graph=g, patterns=[BOOK], mode="count"))
    assert job.applied("local-graph-search")
    pl = make_plan(BOOK, g, rewrite=True)
    want, _ = O.run(g, PL.as_forest(pl), threads=8)
    assert job.counts == want
