"""Seeded input generators shared by tests, the golden-fixture script and
bench.py. Restatements of the reference's generators (pinned against the
reference by tests/golden/make_golden.py):

* ``er`` -- tests/util.py:13-17 of the reference test-suite
* ``powerlaw_edges`` -- cli.gen_synthetic("powerlaw") (cli.py:151-187)
* ``rmat_edges`` -- SURVEY.md A.6 (Graph500 a=.57, b=c=.19, LSB first)
"""
from __future__ import annotations

import numpy as np


def er_edges(n: int, p: float, seed: int, labels: int | None = None):
    rng = np.random.default_rng(seed)
    mask = np.triu(rng.random((n, n)) < p, 1)
    labs = rng.integers(0, labels, n) if labels else None
    return np.argwhere(mask), labs


def er_ref(mod, n, p, seed, labels=None):
    e, labs = er_edges(n, p, seed, labels)
    return mod.from_edges(e, num_vertices=n, labels=labs)


def er(n, p, seed, labels=None):
    from paper_2112_09761_b200 import graph
    return er_ref(graph, n, p, seed, labels)


def complete(n: int, labels=None):
    from paper_2112_09761_b200 import graph
    return graph.from_edges([(a, b) for a in range(n) for b in range(a + 1, n)],
                            num_vertices=n, labels=labels)


def powerlaw_edges(n: int, m: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    targets: list[int] = []
    edges = []
    for v in range(1, n):
        k = min(m, v)
        picked: set[int] = set()
        while len(picked) < k:
            if targets:
                cand = int(targets[rng.integers(0, len(targets))])
            else:
                cand = int(rng.integers(0, v))
            picked.add(cand)
        for w in picked:
            edges.append((v, w))
            targets.extend((v, w))
    return np.asarray(edges, dtype=np.int64).reshape(-1, 2)


def rmat_edges(scale: int, edgefactor: int = 16, seed: int = 1,
               a: float = 0.57, b: float = 0.19, c: float = 0.19) -> np.ndarray:
    rng = np.random.default_rng(seed)
    m = edgefactor << scale
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for bit in range(scale):
        r = rng.random(m)
        ub = r >= ab
        vb = ((r >= a) & (r < ab)) | (r >= abc)
        u |= ub.astype(np.int64) << bit
        v |= vb.astype(np.int64) << bit
    return np.column_stack([u, v])
