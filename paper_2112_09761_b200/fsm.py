"""Bounded-BFS frequent subgraph mining with the level work on the GPU
(reference fsm.py:107-210, ``run_bounded_bfs``; Listing 4).

Semantics are the reference's: edge-induced subgraphs with up to
``max_edges`` edges grow one edge per level; every level's subgraphs are
grouped by quick pattern, then canonical pattern; the support of a pattern is
its minimum-image (domain) support unless a ``support_aggregator`` is given;
patterns the ``pattern_filter`` rejects are pruned together with their
subtrees (domain support is anti-monotone); ``parent_child`` records which
kept pattern produced which; ``blocks_processed`` counts the fixed-capacity
blocks the reference walks (``ExecutionConfig.bfs_block_size``) so the number
is comparable.

Division of work:

* device (``libg2m.so``, ``csrc/fsm_kernels.cuh``): the level-1 edge rows,
  quick-pattern records and their grouping (hash sort + collision check),
  the (pattern, position, vertex) domain triples and their unique runs, the
  parent -> child pairs, and the extension of kept subgraphs by one edge with
  the new edge sets deduplicated (sort by hash, exact compare);
* host: the canonical form of each *distinct* quick pattern (a handful per
  level; k! permutations, k <= 8), the support / filter callbacks, and the
  result dictionaries.
"""
from __future__ import annotations

import ctypes as C
import itertools
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .executor import ExecutionConfig
from .graph import Graph, label_frequency
from .pattern import EDGE_INDUCED, Pattern

MAX_EDGES = 7          # device row layout (kFsmE)
_REC = 12              # quick-record words (kRec)


@dataclass
class SubgraphBlock:
    """One fixed-capacity slice of a BFS level's subgraph list (fsm.py:23-33)."""

    rows: list
    capacity: int

    def __post_init__(self):
        if len(self.rows) > self.capacity:
            raise ValueError("block exceeds its capacity")


def pattern_from_key(key: tuple) -> Pattern:
    k, labels, edges = key
    return Pattern(k, edges, labels=labels, induced=EDGE_INDUCED)


def min_image_support(domains: list[set[int]]) -> int:
    """Minimum over pattern positions of the distinct data vertices mapped
    there (the anti-monotone domain support, fsm.py:88-91)."""
    return min(len(d) for d in domains)


@dataclass
class FsmResult:
    frequent: dict[tuple, int]
    all_supports: dict[tuple, int]
    parent_child: set[tuple[tuple, tuple]]
    blocks_processed: int
    label_pruning: bool

    def frequent_patterns(self) -> dict[Pattern, int]:
        return {pattern_from_key(k): s for k, s in self.frequent.items()}


def canonical_form(labels: tuple[int, ...], pairs: tuple[tuple[int, int], ...]):
    """Canonical key of a labeled pattern given by vertex labels (position
    order) and edges as position pairs, plus every position map that attains
    it (fsm.py:50-80): over all relabellings perm (position i -> perm[i]),
    the lexicographically smallest (labels by new position, sorted edges);
    a map is the inverse permutation (new position -> old position)."""
    k = len(labels)
    best = None
    maps: list[tuple[int, ...]] = []
    for perm in itertools.permutations(range(k)):
        inv = [0] * k
        for old, new in enumerate(perm):
            inv[new] = old
        lab = tuple(labels[inv[c]] for c in range(k))
        if best is not None and lab > best[0]:
            continue
        edg = tuple(sorted((min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in pairs))
        cand = (lab, edg)
        if best is None or cand < best:
            best, maps = cand, [tuple(inv)]
        elif cand == best:
            maps.append(tuple(inv))
    return (k, best[0], best[1]), maps


def _decode_record(rec: np.ndarray):
    k = int(rec[0]) & 0xff
    ne = (int(rec[0]) >> 8) & 0xff
    labels = tuple(int(x) for x in rec[1:1 + k])
    packed = int(rec[9]) | (int(rec[10]) << 32)
    pairs = tuple(((packed >> (6 * e + 3)) & 7, (packed >> (6 * e)) & 7) for e in range(ne))
    return labels, pairs


class _Fsm:
    """Owning handle of the device-side level state (``g2m_fsm``)."""

    def __init__(self, dg, ok: np.ndarray | None):
        self.h = C.c_void_p()
        n = C.c_uint64(0)
        N.check(N.lib().g2m_fsm_create(dg.handle, None if ok is None else N.ptr(ok, C.c_uint8),
                                       C.byref(self.h), C.byref(n)), "fsm create")
        self.n = int(n.value)
        self.level = 1

    def close(self):
        if self.h:
            N.lib().g2m_fsm_destroy(self.h)
            self.h = None

    def rows(self):
        e = np.zeros(self.n * MAX_EDGES, dtype=np.uint64)
        v = np.zeros(self.n * 8, dtype=np.uint32)
        k = np.zeros(self.n, dtype=np.uint8)
        if self.n:
            N.check(N.lib().g2m_fsm_rows(self.h, N.ptr(e, C.c_uint64), N.ptr(v, C.c_uint32),
                                         N.ptr(k, C.c_uint8)), "fsm rows")
        out = []
        for r in range(self.n):
            verts = tuple(int(x) for x in v[r * 8:r * 8 + int(k[r])])
            edges = tuple((int(x >> np.uint64(32)), int(x & np.uint64(0xffffffff)))
                          for x in e[r * MAX_EDGES:r * MAX_EDGES + self.level])
            out.append((verts, edges))
        return out

    def keep(self, mask: np.ndarray):
        n = C.c_uint64(0)
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        N.check(N.lib().g2m_fsm_keep(self.h, N.ptr(m, C.c_uint8), C.byref(n)), "fsm keep")
        self.n = int(n.value)


def run_bounded_bfs(g: Graph, max_edges: int, sigma_min: int,
                    cfg: ExecutionConfig | None = None,
                    support_aggregator=None, pattern_filter=None,
                    subgraph_filter=None, label_pruning: bool = True,
                    device: int | None = None) -> FsmResult:
    """Mine all edge-induced patterns with <= max_edges edges whose support
    passes the pattern filter (default: support >= sigma_min)."""
    if g.labels is None:
        raise ValueError("frequent subgraph mining requires a labeled graph")
    if max_edges < 1:
        raise ValueError("max_edges must be at least 1")
    if max_edges > MAX_EDGES:
        raise ValueError(f"max_edges beyond {MAX_EDGES} is not supported on the device")
    cfg = cfg or ExecutionConfig()
    block = cfg.bfs_block_size
    aggregate = support_aggregator or (lambda key, domains: min_image_support(domains))
    keep_pattern = pattern_filter or (lambda key, support: support >= sigma_min)

    ok = None
    if label_pruning and g.num_vertices:
        good = label_frequency(g).frequent_labels(sigma_min)
        ok = np.isin(g.labels, np.asarray(sorted(good), dtype=g.labels.dtype)).astype(np.uint8)

    dev = N.default_device() if device is None else device
    N.require_device(dev)
    dg = g.device_graph(dev)
    st = _Fsm(dg, ok)
    frequent: dict[tuple, int] = {}
    all_supports: dict[tuple, int] = {}
    parent_child: set[tuple[tuple, tuple]] = set()
    blocks = 0
    canon_memo: dict[tuple, tuple] = {}
    prev_keys: list[tuple] = []
    try:
        if subgraph_filter is not None and st.n:
            st.keep(np.array([bool(subgraph_filter(v, e)) for v, e in st.rows()], dtype=np.uint8))
        level = 1
        while st.n and level <= max_edges:
            lib = N.lib()
            nq = C.c_uint64(0)
            N.check(lib.g2m_fsm_quick(st.h, C.byref(nq)), "fsm quick")
            nq = int(nq.value)
            recs = np.zeros(max(nq, 1) * _REC, dtype=np.uint32)
            N.check(lib.g2m_fsm_quick_records(st.h, N.ptr(recs, C.c_uint32)), "fsm records")
            keys: list[tuple] = []
            key_id: dict[tuple, int] = {}
            canon = np.zeros(max(nq, 1), dtype=np.uint32)
            nmaps = np.zeros(max(nq, 1), dtype=np.uint32)
            map_off = np.zeros(max(nq, 1), dtype=np.uint32)
            blob: list[int] = []
            for q in range(nq):
                quick = _decode_record(recs[q * _REC:(q + 1) * _REC])
                hit = canon_memo.get(quick)
                if hit is None:
                    hit = canon_memo[quick] = canonical_form(*quick)
                key, maps = hit
                if key not in key_id:
                    key_id[key] = len(keys)
                    keys.append(key)
                canon[q] = key_id[key]
                nmaps[q] = len(maps)
                map_off[q] = len(blob)
                for m in maps:
                    blob.extend(m)
            mb = np.asarray(blob or [0], dtype=np.uint8)
            ndom, nruns, npc = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
            N.check(lib.g2m_fsm_domains(st.h, N.ptr(canon, C.c_uint32), N.ptr(nmaps, C.c_uint32),
                                        N.ptr(map_off, C.c_uint32), N.ptr(mb, C.c_uint8), len(blob),
                                        C.byref(ndom), C.byref(nruns), C.byref(npc)), "fsm domains")
            rk = np.zeros(max(nruns.value, 1), dtype=np.uint64)
            rl = np.zeros(max(nruns.value, 1), dtype=np.uint64)
            pc = np.zeros(max(npc.value, 1), dtype=np.uint64)
            dk = np.zeros(max(ndom.value, 1), dtype=np.uint64) if support_aggregator else None
            N.check(lib.g2m_fsm_results(st.h, N.ptr(rk, C.c_uint64), N.ptr(rl, C.c_uint64),
                                        None if dk is None else N.ptr(dk, C.c_uint64),
                                        N.ptr(pc, C.c_uint64)), "fsm results")
            if support_aggregator is None:
                sizes: dict[int, list[int]] = {}
                for key64, ln in zip(rk[:nruns.value].tolist(), rl[:nruns.value].tolist()):
                    sizes.setdefault(key64 >> 4, []).append(ln)
                supports = {keys[c]: aggregate(keys[c], [range(x) for x in sizes[c]])
                            for c in range(len(keys))}
            else:
                doms = {c: [set() for _ in range(keys[c][0])] for c in range(len(keys))}
                for key64 in dk[:ndom.value].tolist():
                    doms[key64 >> 36][(key64 >> 32) & 0xf].add(key64 & 0xffffffff)
                supports = {keys[c]: aggregate(keys[c], doms[c]) for c in range(len(keys))}
            all_supports.update(supports)
            kept = {key for key, s in supports.items() if keep_pattern(key, s)}
            frequent.update({key: supports[key] for key in kept})
            for pair in pc[:npc.value].tolist():
                parent_child.add((prev_keys[pair >> 32], keys[pair & 0xffffffff]))
            blocks += math.ceil(st.n / block)
            if level == max_edges:
                break
            mask = np.array([1 if k in kept else 0 for k in keys] or [0], dtype=np.uint8)
            n = C.c_uint64(0)
            N.check(lib.g2m_fsm_extend(st.h, N.ptr(mask, C.c_uint8), len(keys), C.byref(n)), "fsm extend")
            blocks += math.ceil(st.n / block)
            st.n = int(n.value)
            st.level = level + 1
            prev_keys = keys
            if subgraph_filter is not None and st.n:
                st.keep(np.array([bool(subgraph_filter(v, e)) for v, e in st.rows()], dtype=np.uint8))
            level += 1
    finally:
        st.close()
    return FsmResult(frequent=frequent, all_supports=all_supports, parent_child=parent_child,
                     blocks_processed=blocks, label_pruning=label_pruning)


__all__ = ["FsmResult", "SubgraphBlock", "run_bounded_bfs", "min_image_support", "pattern_from_key",
           "canonical_form"]
