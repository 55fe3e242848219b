"""Sorted-set kernels, exposed with the reference's signatures
(pkg/src/patminer/setops.py:21-90) and executed by the device kernel library
(``g2m_setop_batch``: the same warp-cooperative primitives the generated plan
kernels inline). The ``*_batch`` forms run many cases in one launch; the
single-case forms exist for API parity and tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

VERTEX_DTYPE = np.uint32
_EMPTY = np.empty(0, dtype=VERTEX_DTYPE)

OP_INTERSECT, OP_INTERSECT_COUNT, OP_DIFFERENCE, OP_DIFFERENCE_COUNT = 0, 1, 2, 3


def _pack(lists):
    lens = np.fromiter((len(x) for x in lists), dtype=np.uint64, count=len(lists))
    offs = np.zeros(len(lists) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    vals = (np.concatenate([np.asarray(x, dtype=np.uint32) for x in lists])
            if len(lists) and offs[-1] else np.zeros(1, dtype=np.uint32))
    return np.ascontiguousarray(vals, dtype=np.uint32), offs


def setop_batch(op: int, a_lists, b_lists, bounds=None, device: int | None = None):
    """Run one set operation over many (a, b, bound) cases on the GPU.
    Returns counts (int64) and, for materialising ops, the result lists."""
    n = len(a_lists)
    if len(b_lists) != n:
        raise ValueError("a_lists and b_lists differ in length")
    dev = N.default_device() if device is None else device
    N.require_device(dev)
    av, ao = _pack(a_lists)
    bv, bo = _pack(b_lists)
    bd = np.full(n, -1, dtype=np.int64)
    if bounds is not None:
        for i, b in enumerate(bounds):
            if b is not None:
                bd[i] = int(b)
    out_n = np.zeros(max(n, 1), dtype=np.uint64)
    out_v = np.zeros(max(int(ao[-1]) if n else 0, 1), dtype=np.uint32)
    if n:
        N.check(N.lib().g2m_setop_batch(dev, op, n, N.ptr(av, C.c_uint32), N.ptr(ao, C.c_uint64),
                                        N.ptr(bv, C.c_uint32), N.ptr(bo, C.c_uint64),
                                        N.ptr(bd, C.c_int64), N.ptr(out_n, C.c_uint64),
                                        N.ptr(out_v, C.c_uint32)), "setop")
    counts = out_n[:n].astype(np.int64)
    if op in (OP_INTERSECT, OP_DIFFERENCE):
        return counts, [out_v[int(ao[i]):int(ao[i]) + int(counts[i])].copy() for i in range(n)]
    return counts, None


def bound_list(a: np.ndarray, y: int) -> np.ndarray:
    """Prefix of sorted ``a`` strictly below ``y`` (a view; setops.py:21-23)."""
    return a[: int(np.searchsorted(a, y, side="left"))]


def intersect(a, b, bound: int | None = None) -> np.ndarray:
    _, out = setop_batch(OP_INTERSECT, [a], [b], [bound])
    return out[0] if len(out[0]) else _EMPTY


def intersect_count(a, b, bound: int | None = None) -> int:
    c, _ = setop_batch(OP_INTERSECT_COUNT, [a], [b], [bound])
    return int(c[0])


def difference(a, b, bound: int | None = None) -> np.ndarray:
    _, out = setop_batch(OP_DIFFERENCE, [a], [b], [bound])
    return out[0] if len(out[0]) else _EMPTY


def difference_count(a, b, bound: int | None = None) -> int:
    c, _ = setop_batch(OP_DIFFERENCE_COUNT, [a], [b], [bound])
    return int(c[0])


def contains(a: np.ndarray, x: int) -> bool:
    i = int(np.searchsorted(a, x, side="left"))
    return i < len(a) and int(a[i]) == int(x)
