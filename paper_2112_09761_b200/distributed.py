"""Multi-process (one process per GPU) plumbing for the mining path.

The search shards with no data exchange: the graph is replicated per GPU,
each rank mines its chunked round-robin share of the task list (or of the
source vertices for the LGS / wedge kernels), and the only collective is the
final reduction of the per-pattern counts (reference scheduler.py:1-8,
170-239). Counts are exact integers of up to 128 bits,
so they travel as four 32-bit limbs in int64 lanes: a sum over any
realistic number of ranks cannot overflow a lane, and carries are resolved
after the reduction.

The one path with a real exchange step is the diamond count on the support
kernels: per-edge triangle support is not additive over a source split (the
count is Σ_e C(t_e, 2)), but the support ARRAY is. Each rank adds its
sources' triangles into a device array, one all-reduce (sum) of that array
(4 B per DAG edge: 1 GB at RMAT-24) completes every edge's support, and each
rank sums C(t_e, 2) over its own slot share (``diamond_count``).

``torch.distributed`` is the transport (NCCL on GPUs, gloo on CPU for the
tests).
"""
from __future__ import annotations

LIMBS = 4
_MASK = (1 << 32) - 1


ALPHA = 2     # c = ALPHA * y


def resident_warps(device: int = 0) -> int:
    """y of the paper's chunk rule: warps resident on one GPU at once."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        return int(p.multi_processor_count * p.max_threads_per_multi_processor // 32)
    except Exception:
        return 148 * 64     # B200: 148 SMs x 64 warps


def shard(rank: int, world: int, chunk: int | None = None, device: int = 0):
    """The (rr_chunk, rr_parts, rr_part) triple of this rank's chunked
    round-robin share (scheduler.split_chunked_rr's queue ``rank``) with the
    paper's chunk c = ALPHA * y edge tasks, y = resident warps. The
    source-partitioned kernels split sources instead, by the workload
    estimator (executor.source_spec)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    if world == 1:
        return None
    return (int(chunk) if chunk else ALPHA * resident_warps(device), world, rank)


def to_limbs(v: int) -> list[int]:
    if v < 0 or v >> (32 * LIMBS):
        raise ValueError("count outside [0, 2^128)")
    return [(v >> (32 * i)) & _MASK for i in range(LIMBS)]


def from_limbs(limbs) -> int:
    return sum(int(x) << (32 * i) for i, x in enumerate(limbs))


def allreduce_counts(counts: dict[str, int], group=None, device=None) -> dict[str, int]:
    """Sum per-pattern counts over all ranks (same keys, same order on every
    rank); returns exact Python ints."""
    import torch
    import torch.distributed as dist
    keys = list(counts)
    t = torch.tensor([to_limbs(int(counts[k])) for k in keys], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    rows = t.cpu().tolist()
    return {k: from_limbs(r) for k, r in zip(keys, rows)}


def allreduce_max(x: float, group=None, device=None) -> float:
    """Max over ranks (the step time of a data-parallel job)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class SupportStats:
    """device_ms / kernel_ms / tasks / launches of one distributed diamond step."""

    def __init__(self, device_ms: float, kernel_ms: float, tasks: int, launches: int):
        self.device_ms, self.kernel_ms, self.tasks, self.launches = device_ms, kernel_ms, tasks, launches


def diamond_count(g, rank: int, world: int, device: int = 0, rr=None, group=None,
                  name: str = "diamond"):
    """Diamond count of the symmetric graph g over ``world`` ranks: support
    of the rank's sources (``rr``, the chunked round-robin / estimator share
    of executor.source_spec) into a device array, all-reduce (sum), then
    Σ C(t, 2) over the rank's slot share. Returns this rank's additive share
    of the count ({name: share}; ``allreduce_counts`` gives the total) and
    the step's stats (device time = support + all-reduce + sum, CUDA events
    on the rank's device)."""
    import ctypes as C

    import numpy as np
    import torch

    from . import _native as N
    from . import executor as EX

    dg = g.device_graph(device)
    n = C.c_uint64(0)
    N.check(N.lib().g2m_diamond_support(dg.handle, None, None, C.byref(n), None), "diamond support")
    slots = int(n.value)
    dev = torch.device("cuda", device)
    tsup = torch.zeros(max(slots, 1), dtype=torch.int32, device=dev)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(torch.cuda.current_stream(dev))
    spec = EX.source_spec(rr, family="lgs")
    st = N.RunStats()
    N.check(N.lib().g2m_diamond_support(dg.handle, C.byref(spec), C.c_void_p(tsup.data_ptr()), C.byref(n),
                                        C.byref(st)), "diamond support")
    if world > 1:   # the support kernels' stream is drained when the call returns
        import torch.distributed as dist
        dist.all_reduce(tsup, op=dist.ReduceOp.SUM, group=group)
    torch.cuda.synchronize(dev)
    lo, hi = rank * slots // world, (rank + 1) * slots // world
    words = np.zeros(2, dtype=np.uint64)
    st2 = N.RunStats()
    N.check(N.lib().g2m_support_choose2(dg.handle, C.c_void_p(tsup.data_ptr()), lo, hi,
                                        N.ptr(words, C.c_uint64), C.byref(st2)), "support choose2")
    ev1.record(torch.cuda.current_stream(dev))
    ev1.synchronize()
    share = int(words[0]) | (int(words[1]) << 64)
    return {name: share}, SupportStats(ev0.elapsed_time(ev1), st.kernel_ms + st2.kernel_ms,
                                       int(st.tasks), int(st.launches) + 1)
