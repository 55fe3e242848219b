"""Frequent subgraph mining (bounded BFS, fsm.py:107-210) on the GPU against
golden results written by the reference's own run_bounded_bfs
(tests/golden/make_golden_fsm.py), plus the reference's behavioural tests
(test_executor.py:236-300, test_apps.py:150-185)."""
import ast
import json
from pathlib import Path

import numpy as np
import pytest

import graphs as G
import paper_2112_09761_b200 as pm
from paper_2112_09761_b200 import fsm
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200.executor import ExecutionConfig

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "fsm.json").read_text())


def _graph(gen):
    if gen[0] == "tiny":
        return GR.from_edges(np.array([(0, 1), (1, 2)]), labels=np.array([0, 0, 1]))
    _, n, p, seed, nl = gen
    return G.er(n, p, seed, labels=nl)


def _keys(d):
    return {ast.literal_eval(k): v for k, v in d.items()}


# ---- CPU: canonical forms and containers -------------------------------------

def test_canonical_form_basics():
    # a labeled wedge a-b-c with labels (5, 1, 5): centre position moves last / first
    key, maps = fsm.canonical_form((5, 1, 5), ((0, 1), (1, 2)))
    assert key == (3, (1, 5, 5), ((0, 1), (0, 2)))
    assert sorted(maps) == [(1, 0, 2), (1, 2, 0)]            # the two automorphisms
    key2, _ = fsm.canonical_form((5, 5, 1), ((0, 2), (1, 2)))  # same pattern, other order
    assert key2 == key
    k3, m3 = fsm.canonical_form((0, 0, 0), ((0, 1), (0, 2), (1, 2)))
    assert k3 == (3, (0, 0, 0), ((0, 1), (0, 2), (1, 2))) and len(m3) == 6


def test_subgraph_block_capacity():
    fsm.SubgraphBlock([1, 2], 2)
    with pytest.raises(ValueError, match="capacity"):
        fsm.SubgraphBlock([1, 2, 3], 2)


def test_min_image_support_and_exports():
    assert fsm.min_image_support([{1, 2}, {3}]) == 1
    assert pm.run_bounded_bfs is fsm.run_bounded_bfs and pm.FsmResult is fsm.FsmResult
    p = fsm.pattern_from_key((2, (0, 1), ((0, 1),)))
    assert p.size == 2 and p.num_edges == 1


# ---- GPU: parity with the reference --------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD, ids=[f"{c['gen']}-e{c['max_edges']}-s{c['sigma']}" for c in GOLD])
def test_bounded_bfs_equals_reference(case):
    g = _graph(case["gen"])
    cfg = ExecutionConfig(bfs_block_size=case.get("block", 1 << 20))
    res = fsm.run_bounded_bfs(g, case["max_edges"], case["sigma"], cfg=cfg,
                              label_pruning=case.get("pruning", True))
    assert res.frequent == _keys(case["frequent"])
    assert res.all_supports == _keys(case["all_supports"])
    assert res.parent_child == {(ast.literal_eval(a), ast.literal_eval(b)) for a, b in case["parent_child"]}
    assert res.blocks_processed == case["blocks_processed"]


@pytest.mark.gpu
def test_reference_behaviour():
    tiny = GR.from_edges(np.array([(0, 1), (1, 2)]), labels=np.array([0, 0, 1]))
    assert sorted(fsm.run_bounded_bfs(tiny, 1, 1).frequent.values()) == [1, 2]
    k4 = G.complete(4, labels=np.zeros(4, dtype=np.uint32))
    assert fsm.run_bounded_bfs(k4, 2, 5).frequent == {}
    for seed in (1, 2):
        g = G.er(30, 0.15, seed, labels=5)
        for sigma in (2, 3):
            on = fsm.run_bounded_bfs(g, 3, sigma, label_pruning=True)
            off = fsm.run_bounded_bfs(g, 3, sigma, label_pruning=False)
            assert on.frequent == off.frequent
    g = G.er(32, 0.15, 6, labels=3)
    res = fsm.run_bounded_bfs(g, 3, 2)
    assert res.parent_child
    for parent, child in res.parent_child:
        assert res.all_supports[child] <= res.all_supports[parent]
    with pytest.raises(ValueError):
        fsm.run_bounded_bfs(G.complete(3), 2, 1)
    g = G.er(24, 0.2, 7, labels=3)
    small = fsm.run_bounded_bfs(g, 2, 1, cfg=ExecutionConfig(bfs_block_size=8))
    large = fsm.run_bounded_bfs(g, 2, 1)
    assert small.frequent == large.frequent and small.blocks_processed > large.blocks_processed


@pytest.mark.gpu
def test_hooks():
    g = GR.from_edges(np.array([(0, 1), (1, 2)]), labels=np.array([0, 0, 1]))
    res = fsm.run_bounded_bfs(g, 1, 1, pattern_filter=lambda key, s: s == 2)
    assert list(res.frequent.values()) == [2]
    seen = []
    fsm.run_bounded_bfs(g, 1, 1, support_aggregator=lambda key, doms: (seen.append(key),
                                                                       fsm.min_image_support(doms))[1])
    assert seen
    res = fsm.run_bounded_bfs(g, 1, 1, subgraph_filter=lambda verts, edges: 2 not in verts)
    assert list(res.frequent.values()) == [2]
    # a filter on the growing levels too
    h = G.er(26, 0.2, 3, labels=2)
    a = fsm.run_bounded_bfs(h, 3, 2, subgraph_filter=lambda verts, edges: min(verts) > 2)
    b = fsm.run_bounded_bfs(G.er(26, 0.2, 3, labels=2), 3, 2)
    assert set(a.all_supports) <= set(b.all_supports)


@pytest.mark.gpu
def test_k_fsm_api():
    g = G.complete(4, labels=np.zeros(4, dtype=np.uint32))
    res = pm.k_fsm(g, 1, 4)
    assert list(res.counts.values()) == [4]
    (p,) = res.patterns.values()
    assert p.size == 2 and p.num_edges == 1
    assert pm.k_fsm(g, 2, 5).counts == {}
    assert res.applied("bounded-bfs") and res.applied("label-frequency-pruning")
    assert not pm.k_fsm(g, 1, 1, label_pruning=False).applied("label-frequency-pruning")
    with pytest.raises(ValueError):
        pm.k_fsm(G.complete(4), 2, 1)
    case = next(c for c in GOLD if c["gen"] == ["er", 30, 0.15, 41, 3])
    got = pm.k_fsm(_graph(case["gen"]), 3, 2)
    want = {fsm.pattern_from_key(k).canonical_form(): v for k, v in _keys(case["frequent"]).items()}
    assert {p.canonical_form(): s for p, s in got.fsm.frequent_patterns().items()} == want
