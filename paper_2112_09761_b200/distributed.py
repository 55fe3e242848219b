"""Multi-process (one process per GPU) plumbing for the mining path.

The search shards with no data exchange: the graph is replicated per GPU,
each rank mines its chunked round-robin share of the task list (or of the
source vertices for the LGS / wedge kernels), and the only collective is the
final reduction of the per-pattern counts (reference scheduler.py:1-8,
170-239). Counts are exact integers of up to 128 bits,
so they travel as four 32-bit limbs in int64 lanes: a sum over any
realistic number of ranks cannot overflow a lane, and carries are resolved
after the reduction.

``torch.distributed`` is the transport (NCCL on GPUs, gloo on CPU for the
tests); nothing here touches the kernels.
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
