"""Shared builders (mirrors the reference suite's tests/util.py helpers)."""
from __future__ import annotations

import numpy as np

from graphs import complete, er  # noqa: F401
from paper_2112_09761_b200 import plan as plan_mod
from paper_2112_09761_b200.graph import Graph
from paper_2112_09761_b200.pattern import (GraphStats, Pattern, detect_properties,
                                           enumerate_matching_orders,
                                           generate_symmetry_order, select_matching_order)

DIAMOND_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)]
CYCLE4_EDGES = [(0, 1), (1, 2), (2, 3), (3, 0)]
TAILED_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2)]


def diamond(induced="edge") -> Pattern:
    return Pattern(4, DIAMOND_EDGES, induced=induced)


def cycle4(induced="edge") -> Pattern:
    return Pattern(4, CYCLE4_EDGES, induced=induced)


def analyze(p: Pattern, g=None):
    stats = GraphStats.of(g) if g is not None else None
    mo = select_matching_order(enumerate_matching_orders(p), stats)
    return mo, generate_symmetry_order(p, mo)


def make_plan(p: Pattern, g=None, mode: str = "count", granularity: str = "edge",
              oriented: bool = False, rewrite: bool = False):
    mo, so = analyze(p, g)
    pl = plan_mod.build_plan(p, mo, so, mode, granularity=granularity, oriented=oriented)
    if rewrite:
        pl = plan_mod.apply_counting_rewrite(pl, detect_properties(p, mo, so))
    return pl


def orient_host(g: Graph) -> Graph:
    """Host restatement of graph.orient (reference graph.py:204-221), used
    only to feed the CPU oracle in tests."""
    n = g.num_vertices
    src = np.repeat(np.arange(n, dtype=np.int64), g.degrees)
    dst = g.neighbors.astype(np.int64)
    du, dv = g.degrees[src], g.degrees[dst]
    keep = (du < dv) | ((du == dv) & (src < dst))
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(np.bincount(src[keep], minlength=n), out=off[1:])
    return Graph(off, g.neighbors[keep], labels=g.labels, oriented=True)
