"""Python side of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Serialises a plan forest into oracle.c's node table and runs the C
restatement of the reference executor (executor.py:113-325) over explicit
tasks. Imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

MAXL, MAXP, MAXC = 9, 32, 24
_ACT = {"descend": 0, "emit_count": 1, "binomial_count": 2, "emit_match": 3}


class ONode(C.Structure):
    _fields_ = [("level", C.c_int), ("base_kind", C.c_int), ("base_ref", C.c_int),
                ("ni", C.c_int), ("inter", C.c_int * MAXL),
                ("ns", C.c_int), ("sub", C.c_int * MAXL),
                ("label", C.c_int), ("buffered", C.c_int),
                ("nchild", C.c_int), ("child", C.c_int * MAXC),
                ("members", C.c_uint32),
                ("bound", C.c_int * MAXP), ("action", C.c_int * MAXP), ("tail", C.c_int * MAXP)]


_lib = None


def build() -> Path:
    """Compile oracle.c into oracle/_build/liboracle.so (gcc)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.oracle_run.restype = C.c_int
        L.oracle_run.argtypes = [
            C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.c_uint64,
            C.c_uint64, C.POINTER(ONode), C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int,
            C.c_int, C.POINTER(C.c_int64), C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
            C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.c_uint64, C.c_int,
            C.POINTER(C.c_uint64)]
        L.oracle_node_size.restype = C.c_int
        assert L.oracle_node_size() == C.sizeof(ONode), "oracle node layout mismatch"
        _lib = L
    return _lib


def serialize(forest):
    """PlanForest -> (node table, root indices, pattern ids)."""
    pids = list(forest.pattern_ids)
    pidx = {p: i for i, p in enumerate(pids)}
    nodes: list[ONode] = []

    def add(node) -> int:
        me = len(nodes)
        nd = ONode()
        nodes.append(nd)
        nd.level = node.level
        kind = node.expr.base[0]
        nd.base_kind = {"universe": 0, "nbr": 1, "buf": 2}[kind]
        nd.base_ref = node.expr.base[1] if kind != "universe" else 0
        nd.ni = len(node.expr.intersect)
        for i, j in enumerate(node.expr.intersect):
            nd.inter[i] = j
        nd.ns = len(node.expr.subtract)
        for i, j in enumerate(node.expr.subtract):
            nd.sub[i] = j
        nd.label = -1 if node.expr.label is None else int(node.expr.label)
        nd.buffered = int(bool(node.buffered))
        m = 0
        for p in node.members:
            m |= 1 << pidx[p]
        nd.members = m
        for p in range(MAXP):
            nd.bound[p] = -1
        for p, b in node.bounds.items():
            nd.bound[pidx[p]] = -1 if b is None else int(b)
        for p, (a, t) in node.actions.items():
            nd.action[pidx[p]] = _ACT[a]
            nd.tail[pidx[p]] = int(t)
        kids = [add(c) for c in node.children]
        if len(kids) > MAXC:
            raise ValueError("too many children for the oracle node table")
        nodes[me].nchild = len(kids)
        for i, k in enumerate(kids):
            nodes[me].child[i] = k
        return me

    roots = [add(r) for r in forest.roots]
    arr = (ONode * len(nodes))(*nodes)
    return arr, (C.c_int * len(roots))(*roots), pids


def _edge_pairs(g, reduced: bool) -> np.ndarray:
    off = np.asarray(g.row_offsets, dtype=np.int64)
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(off))
    arr = np.column_stack([src, np.asarray(g.neighbors, dtype=np.int64)])
    if reduced:
        arr = arr[arr[:, 0] > arr[:, 1]]
    return np.ascontiguousarray(arr)


def default_tasks(g, forest) -> tuple[bool, np.ndarray]:
    """The reference's default task list for a forest (executor.py:355-367)."""
    plans = list(forest.plans.values())
    if forest.parallel_granularity == "edge":
        reduced = (not g.oriented) and all(pl.constrains_first_edge() for pl in plans)
        return True, _edge_pairs(g, reduced)
    return False, np.arange(g.num_vertices, dtype=np.int64)


def run(g, forest, tasks=None, edge: bool | None = None, threads: int | None = None,
        list_cap: int = 0):
    """Counts (dict pid -> int), algorithmic bytes (int) and optionally the
    match stream [(pid, tuple)] of a forest on graph g (host arrays)."""
    nodes, roots, pids = serialize(forest)
    if tasks is None:
        edge, tasks = default_tasks(g, forest)
    tasks = np.ascontiguousarray(tasks, dtype=np.int64)
    if edge is None:
        edge = tasks.ndim == 2
    ntasks = len(tasks)
    off = np.ascontiguousarray(g.row_offsets, dtype=np.uint64)
    nbr = np.ascontiguousarray(g.neighbors, dtype=np.uint32)
    if len(nbr) == 0:
        nbr = np.zeros(1, dtype=np.uint32)
    lab = None if g.labels is None else np.ascontiguousarray(g.labels, dtype=np.uint32)
    counts = np.zeros(2 * max(len(pids), 1), dtype=np.uint64)
    nbytes = np.zeros(2, dtype=np.uint64)
    width = max(pl.depth for pl in forest.plans.values()) + 1
    mout = np.zeros(max(list_cap, 1) * width, dtype=np.uint32) if list_cap else None
    mcount = C.c_uint64(0)
    nthreads = threads or os.cpu_count() or 1
    rc = lib().oracle_run(
        off.ctypes.data_as(C.POINTER(C.c_uint64)), nbr.ctypes.data_as(C.POINTER(C.c_uint32)),
        None if lab is None else lab.ctypes.data_as(C.POINTER(C.c_uint32)),
        g.num_vertices, max(int(g.max_degree), 1), nodes, len(nodes), roots, len(roots),
        len(pids), int(bool(edge)),
        tasks.ctypes.data_as(C.POINTER(C.c_int64)) if ntasks else None, ntasks, nthreads,
        counts.ctypes.data_as(C.POINTER(C.c_uint64)), nbytes.ctypes.data_as(C.POINTER(C.c_uint64)),
        None if mout is None else mout.ctypes.data_as(C.POINTER(C.c_uint32)), list_cap, width,
        C.byref(mcount))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    out = {p: int(counts[2 * i]) | (int(counts[2 * i + 1]) << 64) for i, p in enumerate(pids)}
    alg = int(nbytes[0]) | (int(nbytes[1]) << 64)
    if mout is None:
        return out, alg
    stream = []
    depth = {p: forest.plans[p].depth for p in pids}
    for i in range(min(int(mcount.value), list_cap)):
        row = mout[i * width:(i + 1) * width]
        p = pids[int(row[0])]
        stream.append((p, tuple(int(x) for x in row[1:1 + depth[p]])))
    return out, alg, stream
