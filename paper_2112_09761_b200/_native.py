"""ctypes binding of libg2m.so (the C ABI declared in include/g2m.h).

This is the only module that touches the native library. There is no CPU
fallback: if the library is missing, or no CUDA device is visible, the
mining entry points raise instead of computing anything on the host.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libg2m.so"
DEVICE_HEADER = PKG_DIR / "csrc" / "g2m_device.cuh"

ABI_VERSION = 7                     # G2M_ABI_VERSION in include/g2m.h
G2M_OK, G2M_EUSAGE, G2M_EBUDGET, G2M_ECUDA, G2M_STOPPED = 0, 1, 2, 3, 4
TASKS_EDGE, TASKS_VERTEX = 0, 1
SRC_IMPLICIT, SRC_PAIRS, SRC_VERTICES, SRC_INDEX = 0, 1, 2, 3


class GraphInfo(C.Structure):
    _fields_ = [("num_vertices", C.c_uint64), ("num_slots", C.c_uint64),
                ("max_degree", C.c_uint64), ("oriented", C.c_int32),
                ("labeled", C.c_int32), ("device", C.c_int32), ("reserved", C.c_int32),
                ("sum_degree_sq", C.c_uint64)]


class TaskSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("source", C.c_int32), ("reduced", C.c_int32),
                ("weighted", C.c_int32), ("data", C.POINTER(C.c_int64)),
                ("count", C.c_uint64), ("rr_chunk", C.c_uint64),
                ("rr_parts", C.c_uint32), ("rr_part", C.c_uint32)]


class KernelMeta(C.Structure):
    _fields_ = [("num_patterns", C.c_int32), ("num_slots", C.c_int32),
                ("granularity", C.c_int32), ("max_level", C.c_int32),
                ("needs_labels", C.c_int32), ("list_mode", C.c_int32),
                ("smem_slot_cap", C.c_int32), ("warps_per_block", C.c_int32),
                ("instrumented", C.c_int32), ("warp_words", C.c_int32),
                ("reserved", C.c_int32 * 6)]


class RunConfig(C.Structure):
    _fields_ = [("blocks", C.c_int32), ("reserved0", C.c_int32), ("chunk", C.c_uint64),
                ("scratch_budget", C.c_uint64), ("time_kernel", C.c_int32),
                ("reserved", C.c_int32 * 5)]


class RunStats(C.Structure):
    _fields_ = [("tasks", C.c_uint64), ("tasks_active", C.c_uint64), ("warps", C.c_uint64),
                ("alg_bytes_lo", C.c_uint64), ("alg_bytes_hi", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("high_water", C.c_uint64 * 8), ("kernel_ms", C.c_double),
                ("total_ms", C.c_double), ("device_ms", C.c_double),
                ("launches", C.c_uint64)]

    @property
    def alg_bytes(self) -> int:
        return int(self.alg_bytes_lo) | (int(self.alg_bytes_hi) << 64)


MATCH_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_uint64,
                       C.POINTER(C.c_uint32))

_P = C.c_void_p
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)

# every symbol include/g2m.h declares, with its ctypes signature
SIGNATURES = {
    "g2m_last_error": (C.c_char_p, []),
    "g2m_abi_version": (C.c_int32, []),
    "g2m_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "g2m_graph_create": (C.c_int, [C.c_int32, _u64p, C.c_uint64, _u32p, C.c_uint64, _u32p,
                                   C.c_int32, C.POINTER(_P)]),
    "g2m_graph_from_edges": (C.c_int, [C.c_int32, _i64p, C.c_uint64, C.c_uint64, _u32p,
                                       C.POINTER(_P)]),
    "g2m_graph_rmat": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                 C.c_double, C.POINTER(_P)]),
    "g2m_graph_orient": (C.c_int, [_P, C.POINTER(_P)]),
    "g2m_graph_replicate": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "g2m_graph_info_get": (C.c_int, [_P, C.POINTER(GraphInfo)]),
    "g2m_graph_download": (C.c_int, [_P, _u64p, _u32p, _u32p]),
    "g2m_graph_destroy": (C.c_int, [_P]),
    "g2m_graph_reduced_tasks": (C.c_int, [_P, _u64p]),
    "g2m_graph_rank_copy": (C.c_int, [_P, C.POINTER(_P)]),
    "g2m_graph_hub_part": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.POINTER(_P), _u64p, _u64p]),
    "g2m_graph_local_ids": (C.c_int, [_P, _u32p]),
    "g2m_fsm_create": (C.c_int, [_P, C.POINTER(C.c_uint8), C.POINTER(_P), _u64p]),
    "g2m_fsm_destroy": (C.c_int, [_P]),
    "g2m_fsm_rows": (C.c_int, [_P, _u64p, _u32p, C.POINTER(C.c_uint8)]),
    "g2m_fsm_keep": (C.c_int, [_P, C.POINTER(C.c_uint8), _u64p]),
    "g2m_fsm_quick": (C.c_int, [_P, _u64p]),
    "g2m_fsm_quick_records": (C.c_int, [_P, _u32p]),
    "g2m_fsm_domains": (C.c_int, [_P, _u32p, _u32p, _u32p, C.POINTER(C.c_uint8), C.c_uint64, _u64p, _u64p,
                                  _u64p]),
    "g2m_fsm_results": (C.c_int, [_P, _u64p, _u64p, _u64p, _u64p]),
    "g2m_fsm_extend": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_uint32, _u64p]),
    "g2m_kernel_work": (C.c_int, [_P, C.c_int32, _u64p]),
    "g2m_kernel_compile": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p),
                                     C.POINTER(C.c_char_p), C.c_int32,
                                     C.POINTER(KernelMeta), C.POINTER(_P)]),
    "g2m_kernel_get_meta": (C.c_int, [_P, C.POINTER(KernelMeta)]),
    "g2m_kernel_destroy": (C.c_int, [_P]),
    "g2m_run": (C.c_int, [_P, _P, C.POINTER(TaskSpec), C.POINTER(RunConfig), _u64p,
                          C.POINTER(RunStats)]),
    "g2m_list": (C.c_int, [_P, _P, C.POINTER(TaskSpec), C.POINTER(RunConfig), MATCH_CB,
                           C.c_void_p, _u64p, C.POINTER(RunStats)]),
    "g2m_run_bfs": (C.c_int, [_P, _P, _P, C.POINTER(TaskSpec), C.POINTER(RunConfig), C.c_uint32,
                              C.c_uint64, _u64p, C.POINTER(RunStats)]),
    "g2m_clique_count": (C.c_int, [_P, C.c_int32, C.POINTER(TaskSpec), _P, C.POINTER(RunConfig),
                                   _u64p, C.POINTER(RunStats)]),
    "g2m_cycle4_count": (C.c_int, [_P, C.POINTER(TaskSpec), C.POINTER(RunConfig), _u64p,
                                   C.POINTER(RunStats)]),
    "g2m_diamond_count": (C.c_int, [_P, C.POINTER(RunConfig), _u64p, C.POINTER(RunStats)]),
    "g2m_diamond_support": (C.c_int, [_P, C.POINTER(TaskSpec), C.c_void_p, _u64p, C.POINTER(RunStats)]),
    "g2m_support_choose2": (C.c_int, [_P, C.c_void_p, C.c_uint64, C.c_uint64, _u64p,
                                      C.POINTER(RunStats)]),
    "g2m_setop_batch": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, _u32p, _u64p, _u32p,
                                  _u64p, _i64p, _u64p, _u32p]),
}

_lib = None
_lib_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """libg2m.so is missing or no CUDA device is visible (no CPU fallback)."""


def load_library():
    """Load libg2m.so (symbols only; does not require a GPU)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.g2m_abi_version() != ABI_VERSION:
                raise NativeUnavailable(f"{LIB_PATH} has ABI {lib.g2m_abi_version()}, "
                                        f"this package needs {ABI_VERSION}; rebuild it")
            _lib = lib
    return _lib


def lib():
    return load_library()


def last_error() -> str:
    msg = lib().g2m_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> int:
    if rc in (G2M_OK, G2M_STOPPED):
        return rc
    msg = last_error()
    if rc == G2M_EUSAGE:
        raise ValueError(msg)
    if rc == G2M_EBUDGET:
        from .executor import BudgetError
        raise BudgetError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


_devcount = None


def device_count() -> int:
    global _devcount
    if _devcount is None:
        n = C.c_int32(0)
        rc = lib().g2m_device_count(C.byref(n))
        _devcount = int(n.value) if rc == G2M_OK else 0
    return _devcount


def require_device(device: int = 0) -> None:
    n = device_count()
    if n <= device:
        raise NativeUnavailable(
            f"CUDA device {device} not available ({n} visible): the B200 engine has no CPU path")


def ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def header_sources() -> tuple[list[bytes], list[bytes]]:
    return [DEVICE_HEADER.read_bytes()], [b"g2m_device.cuh"]


def default_device() -> int:
    return int(os.environ.get("G2M_DEVICE", "0"))
