"""Execution operators: ``run_dfs`` and ``run_dfs_lgs`` on the B200.

Same signatures, validation, errors and result types as the reference
executor (pkg/src/patminer/executor.py:37-106, 339-408, 526-599); the work
itself is one generated sm_100a kernel per plan forest (``codegen.py``),
compiled by NVRTC inside libg2m.so and launched through the C ABI
(``g2m_run`` / ``g2m_list``). There is no host execution path: without the
native library or a visible GPU these functions raise.

"Workers" keep the reference's meaning for reporting and for the memory
budget formula (``resolve_worker_count``, executor.py:47-62); on the device
the unit of parallelism is a resident warp.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from . import codegen, codegen_lgs
from .graph import EdgeTaskList, Graph, build_edge_tasks
from .pattern import EDGE_INDUCED
from .plan import (EDGE_PARALLEL, EMIT_MATCH, VERTEX_PARALLEL, PlanForest,
                   SearchPlan, as_forest, emit_source, iter_nodes)

ID_WIDTH = 4  # bytes per vertex id in the worker-budget formula


class BudgetError(RuntimeError):
    """Memory budget cannot fit even a single worker's scratch."""


class StopSearch(Exception):
    """A match sink requested early termination (kept for API parity)."""


@dataclass
class ExecutionConfig:
    granularity: str = EDGE_PARALLEL
    workers: int = 1
    memory_budget: int | None = None     # bytes available for worker scratch
    lgs: str = "auto"                    # local graph search: auto | on | off
    lgs_delta_threshold: int = 1024
    bfs_block_size: int = 1 << 20
    search: str = "auto"                 # dfs | bfs | auto (bounded-frontier BFS chooser)
    bfs_chunk: int = 32                  # level-3 candidates per frontier item
    frontier_bytes: int | None = None    # frontier buffer bound (None: FRONTIER_BUDGET)


def resolve_worker_count(cfg: ExecutionConfig, num_buffers: int,
                         max_degree: int, num_tasks: int) -> int:
    """min(Y // (X * max_degree * 4), tasks) under a budget Y, else the
    requested count, clamped to >= 1 (executor.py:47-62)."""
    if cfg.memory_budget is not None:
        unit = max(num_buffers, 1) * max(max_degree, 1) * ID_WIDTH
        cap = cfg.memory_budget // unit
        if cap < 1:
            raise BudgetError(f"budget {cfg.memory_budget} B < one worker's scratch ({unit} B)")
        return max(1, min(int(cap), num_tasks))
    return max(1, min(cfg.workers, max(num_tasks, 1)))


class WorkerContext:
    """Per-worker counters (executor.py:65-81). On the GPU a worker's scratch
    is a warp's slots; this host object remains for API compatibility and
    for merging per-device results."""

    def __init__(self, num_buffers: int, capacity: int, pattern_ids, sink=None):
        self.scratch = [np.empty(max(capacity, 1), dtype=np.uint32) for _ in range(num_buffers)]
        self.high_water = [0] * num_buffers
        self.counts: dict[str, int] = {pid: 0 for pid in pattern_ids}
        self.sink = sink
        self.tasks_done = 0


def merge_results(contexts: list[WorkerContext]) -> dict[str, int]:
    total: dict[str, int] = {}
    for ctx in contexts:
        for pid, c in ctx.counts.items():
            total[pid] = total.get(pid, 0) + c
    return total


@dataclass
class ExecStats:
    workers: int
    tasks: int
    num_buffers: int
    buffer_high_water: tuple[int, ...]
    elapsed_s: float
    kernel_ms: float = 0.0
    device: int = 0
    gpu_warps: int = 0


@dataclass
class RunResult:
    counts: dict[str, int]
    stats: ExecStats
    stopped_early: bool = False


# ---------------------------------------------------------------------------
# kernel cache
# ---------------------------------------------------------------------------

WARPS_PER_BLOCK = 8
# Per-warp shared memory of the generated kernel (u32 words): materialised-set
# slots live in shared memory only when they fit SMEM_SLOT_WORDS (otherwise a
# global slab), loop-invariant lists are staged up to STAGE_WORDS. Smaller
# footprints buy occupancy: 4-motif power-law 200k 90.6 -> 55.3 ms going
# from 4096/1024 to global slots + 256 (profiles/r02/mc4_occupancy.txt).
SMEM_SLOT_WORDS = int(os.environ.get("G2M_SMEM_SLOT_WORDS", 1024))
STAGE_WORDS = int(os.environ.get("G2M_STAGE_WORDS", 256))


class CompiledPlan:
    """A generated kernel compiled for sm_100a (owned ``g2m_kernel``)."""

    def __init__(self, gen: codegen.GeneratedKernel, handle: int, compile_s: float):
        self.gen = gen
        self.handle = handle
        self.compile_s = compile_s

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h and N._lib is not None:
            try:
                N._lib.g2m_kernel_destroy(h)
            except Exception:
                pass


_cache: dict[str, CompiledPlan] = {}
_cache_lock = threading.Lock()


def _slot_capacity(forest: PlanForest, labeled: bool, max_degree: int) -> int:
    slots = codegen.slots_needed(forest, labeled)
    if slots == 0:
        return 0
    cap = 64
    while cap < max_degree:
        cap *= 2
    if slots * cap <= SMEM_SLOT_WORDS:
        return cap
    return 0


def compile_forest(forest: PlanForest, labeled: bool, list_mode: bool, max_degree: int,
                   flatten: bool = True, instrument: bool = False,
                   frontier: str | None = None) -> CompiledPlan:
    """Generate + NVRTC-compile (cached by generated source)."""
    cap = _slot_capacity(forest, labeled, max_degree)
    gen = codegen.generate(forest, labeled=labeled, list_mode=list_mode,
                           smem_slot_cap=cap, warps_per_block=WARPS_PER_BLOCK,
                           stage_words=STAGE_WORDS, flatten=flatten, instrument=instrument,
                           frontier=frontier)
    return _compile_gen(gen, instrument)


def _compile_gen(gen: codegen.GeneratedKernel, instrument: bool) -> CompiledPlan:
    key = gen.key
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            return hit
        meta = N.KernelMeta()
        meta.num_patterns = gen.num_patterns
        meta.num_slots = gen.num_slots
        meta.granularity = gen.granularity
        meta.max_level = gen.max_level
        meta.needs_labels = int(gen.labeled)
        meta.list_mode = int(gen.list_mode)
        meta.smem_slot_cap = gen.smem_slot_cap
        meta.warps_per_block = gen.warps_per_block
        meta.warp_words = gen.warp_words
        meta.instrumented = int(instrument)
        hsrc, hnames = N.header_sources()
        arr_src = (C.c_char_p * len(hsrc))(*hsrc)
        arr_names = (C.c_char_p * len(hnames))(*hnames)
        h = C.c_void_p()
        t0 = time.perf_counter()
        N.check(N.lib().g2m_kernel_compile(gen.source.encode(), gen.name.encode(), arr_src,
                                           arr_names, len(hsrc), C.byref(meta), C.byref(h)),
                "kernel compile")
        cp = CompiledPlan(gen, h.value, time.perf_counter() - t0)
        _cache[key] = cp
        return cp


# ---------------------------------------------------------------------------
# task specs
# ---------------------------------------------------------------------------

class VertexTasks:
    """The implicit vertex task list ``arange(|V|)`` (executor.py:365-366)."""

    def __init__(self, n: int):
        self.n = n

    def __len__(self) -> int:
        return self.n

    def __array__(self, dtype=None, copy=None):
        return np.arange(self.n, dtype=dtype or np.int64)


def task_spec(tasks, *, rr=None, index: np.ndarray | None = None):
    """Build a ``g2m_task_spec``; returns (spec, keepalive array)."""
    spec = N.TaskSpec()
    keep = None
    if isinstance(tasks, EdgeTaskList):
        spec.kind = N.TASKS_EDGE
        spec.reduced = int(bool(tasks.reduced))
        if index is not None:
            if not tasks.is_implicit:
                keep = np.ascontiguousarray(tasks.edges[index], dtype=np.int64)
                spec.source = N.SRC_PAIRS
                spec.count = len(keep)
            else:
                keep = np.ascontiguousarray(index, dtype=np.int64)
                spec.source = N.SRC_INDEX
                spec.count = len(keep)
        elif tasks.is_implicit:
            spec.source = N.SRC_IMPLICIT
        else:
            keep = np.ascontiguousarray(tasks.edges, dtype=np.int64).reshape(-1, 2)
            spec.source = N.SRC_PAIRS
            spec.count = len(keep)
    else:
        spec.kind = N.TASKS_VERTEX
        if isinstance(tasks, VertexTasks) and index is None:
            spec.source = N.SRC_IMPLICIT
        else:
            arr = np.asarray(tasks, dtype=np.int64).reshape(-1)
            if index is not None:
                arr = arr[index]
            keep = np.ascontiguousarray(arr)
            spec.source = N.SRC_VERTICES
            spec.count = len(keep)
    if rr is not None:
        spec.rr_chunk, spec.rr_parts, spec.rr_part = rr
    if keep is not None and len(keep):
        spec.data = keep.ctypes.data_as(C.POINTER(C.c_int64))
    return spec, keep


def algorithmic_bytes(g: Graph, forest, tasks=None, device: int | None = None) -> int:
    """SURVEY.md 8(d) algorithmic bytes of the reference plan over `tasks`,
    from an instrumented variant of the generated kernel (not timed)."""
    forest = as_forest(forest)
    if tasks is None:
        tasks = _default_tasks(g, forest)
    _, st, _, _ = execute(g, forest, tasks, device=device, instrument=True)
    return st.alg_bytes


def _counts_from(words: np.ndarray, pids) -> dict[str, int]:
    out = {}
    for i, pid in enumerate(pids):
        out[pid] = int(words[2 * i]) | (int(words[2 * i + 1]) << 64)
    return out


# k values routed to the bitmap local-graph clique kernels (g2m_clique_count);
# G2M_TC_LGS=0 sends triangle counting to the generated plan kernel instead
LGS_CLIQUE_K = {3, 4, 5}
# G2M_LGS_GENERATED=1: run_dfs_lgs sends k-clique counts to the generated
# LGS kernel too (tests compare it with the hand-written tiers)
LGS_GENERATED_CLIQUES = os.environ.get("G2M_LGS_GENERATED") == "1"
if os.environ.get("G2M_TC_LGS") == "0":
    LGS_CLIQUE_K.discard(3)


def _lgs_clique_k(g: Graph, forest: PlanForest, tasks, sink, index) -> int:
    """k if this run can use the bitmap clique kernels, else 0: a single
    count-only clique plan on an oriented, unlabeled graph over its implicit
    (whole or round-robin) task list."""
    if len(forest.plans) != 1 or index is not None or g.labels is not None:
        return 0
    pl = forest.single()
    p = pl.pattern
    if not (p.is_clique() and pl.uses_orientation and g.oriented and p.labels is None):
        return 0
    if sink is not None and pl.mode == "list":
        return 0
    if not (isinstance(tasks, EdgeTaskList) and tasks.is_implicit):
        return 0
    return p.size if p.size in LGS_CLIQUE_K else 0


def _is_cycle4_count(g: Graph, forest: PlanForest, tasks, sink, index) -> bool:
    """A single count-only, unlabeled, edge-induced 4-cycle plan on a
    symmetric graph over its implicit (whole or round-robin) task list: the
    wedge-aggregation kernels (g2m_cycle4_count) give the same count."""
    if len(forest.plans) != 1 or index is not None or g.labels is not None or g.oriented:
        return False
    pl = forest.single()
    p = pl.pattern
    if not (p.size == 4 and len(p.edges) == 4 and all(p.degree(v) == 2 for v in range(4))):
        return False
    if p.induced != EDGE_INDUCED or p.labels is not None or pl.uses_orientation:
        return False
    if sink is not None and pl.mode == "list":
        return False
    if isinstance(tasks, EdgeTaskList):
        return tasks.is_implicit
    return isinstance(tasks, VertexTasks)


def _is_diamond_count(g: Graph, forest: PlanForest, tasks, sink, index, rr) -> bool:
    """A single count-only, unlabeled, edge-induced diamond plan on a
    symmetric graph over its whole implicit task list (one device): the
    edge triangle-support kernels (g2m_diamond_count) give the same count."""
    if len(forest.plans) != 1 or index is not None or rr is not None:
        return False
    if g.labels is not None or g.oriented:
        return False
    pl = forest.single()
    p = pl.pattern
    if not (p.size == 4 and len(p.edges) == 5
            and sorted(p.degree(v) for v in range(4)) == [2, 2, 3, 3]):
        return False
    if p.induced != EDGE_INDUCED or p.labels is not None or pl.uses_orientation:
        return False
    if sink is not None and pl.mode == "list":
        return False
    if isinstance(tasks, EdgeTaskList):
        return tasks.is_implicit
    return isinstance(tasks, VertexTasks)


# How the source-partitioned kernels (bitmap k-clique, 4-cycle wedges) split
# their sources over the parts of a multi-GPU run: "est" = the pattern-aware
# workload estimator (runs of consecutive rank-space sources of equal
# estimated work, SOURCE_CHUNK sources per run on average, dealt round-robin;
# PAPER.md:1256-1262, 1309-1322), "rr" = sources dealt one by one in rank
# order. Chunk per family from the 8-part simulation on one B200
# (profiles/r02/sim_*.json, max/mean kernel time over the parts):
#   bitmap k-clique RMAT-22:  est:16  1.050 (4-clique) 1.035 (TC); est:256 2.21 / 1.11; rr:1 1.057 / 1.034
#   4-cycle wedges RMAT-24:   est:256 1.017; est:16 1.067; rr:1 1.005
# G2M_SOURCE_SPLIT=est[:c] | rr overrides both.
SOURCE_SPLIT = "est"
SOURCE_CHUNK = {"lgs": 16, "cycle4": 256}
_ss = os.environ.get("G2M_SOURCE_SPLIT")
if _ss:
    SOURCE_SPLIT, _, _c = _ss.partition(":")
    if _c:
        SOURCE_CHUNK = {"lgs": int(_c), "cycle4": int(_c)}


def source_spec(rr, split: str | None = None, chunk: int | None = None,
                family: str = "lgs") -> N.TaskSpec:
    """The vertex-partition spec of a source-partitioned kernel for the
    part rr = (c, n, i) of a chunked round-robin schedule (None: all
    sources). The edge-task chunk c does not apply: the parts split the
    *sources* (whose weights differ by orders of magnitude), either by the
    workload estimator or one by one."""
    spec = N.TaskSpec()
    spec.kind = N.TASKS_VERTEX
    if rr is None:
        return spec
    split = split or SOURCE_SPLIT
    if split == "est":
        spec.rr_chunk, spec.weighted = int(chunk or SOURCE_CHUNK[family]), 1
    elif split == "rr":
        spec.rr_chunk = int(chunk or 1)
    else:
        raise ValueError(f"unknown source split {split!r}")
    spec.rr_parts, spec.rr_part = int(rr[1]), int(rr[2])
    return spec


def kernel_family(g: Graph, forest: PlanForest, tasks, sink=None, index=None, rr=None,
                  lgs: bool = True, instrument: bool = False) -> str:
    """Which kernels ``execute`` runs for this forest: "lgs" (bitmap k-clique),
    "cycle4" (wedge aggregation), "diamond" (edge triangle support) or
    "plan" (the generated plan kernel, DFS or bounded BFS)."""
    if instrument or not lgs:
        return "plan"
    if _lgs_clique_k(g, forest, tasks, sink, index):
        return "lgs"
    if _is_cycle4_count(g, forest, tasks, sink, index):
        return "cycle4"
    if _is_diamond_count(g, forest, tasks, sink, index, rr):
        return "diamond"
    return "plan"


def _skewed(g: Graph) -> bool:
    avg = g.num_edges / max(g.num_vertices, 1)
    return g.max_degree >= SKEW_FOR_BFS * max(avg, 1.0)


def _edge_form(forest: PlanForest) -> PlanForest:
    """The same forest with edge-parallel task granularity (plans are
    identical apart from the granularity tag, plan.py:110-174)."""
    plans = {pid: replace(pl, parallel_granularity=EDGE_PARALLEL) for pid, pl in forest.plans.items()}
    return replace(forest, plans=plans, parallel_granularity=EDGE_PARALLEL)


FRONTIER_BUDGET = 16 << 30      # bytes of level-3 frontier items kept in HBM at once
FRONTIER_ITEM = 16              # bytes per item (G2MItem)
SKEW_FOR_BFS = 8.0              # max degree / average degree that makes DFS lopsided


def frontier_estimate(g: Graph, forest: PlanForest, tasks, chunk: int) -> int:
    """Upper bound (bytes) of the level-3 frontier of the BFS runtime:
    nodes3 * (Σ_tasks d(v1) / chunk + tasks) items, Σ_tasks d(v1) <= Σ_v d(v)^2."""
    n3 = codegen.frontier_nodes(forest)
    items = n3 * (float(g.sum_degree_sq()) / max(chunk, 1) + len(tasks))
    return int(items * FRONTIER_ITEM)


def choose_search(g: Graph, forest: PlanForest, tasks, cfg: ExecutionConfig | None = None,
                  sink=None) -> tuple[str, str]:
    """DFS or bounded-frontier BFS for one forest on one graph, with the
    reason (the "bounded-bfs" optimisation-log line). BFS needs a level-3
    node with children to split (edge-parallel count forests, unlabeled);
    ``auto`` takes it when the degree distribution is skewed enough for
    warp-per-edge DFS to be lopsided and the whole level-3 frontier fits the
    budget: items <= nodes3 * (Σ_tasks d(v1) / chunk + tasks) with
    Σ_tasks d(v1) <= Σ_v d(v)^2 (SURVEY A.5 sizes it exactly for 4-motifs)."""
    cfg = cfg or ExecutionConfig()
    mode = cfg.search
    if mode not in ("auto", "dfs", "bfs"):
        raise ValueError(f"unknown search strategy {mode!r}")
    n3 = codegen.frontier_nodes(forest)
    if mode == "dfs":
        return "dfs", "depth-first search requested"
    if n3 == 0 or not isinstance(tasks, EdgeTaskList) or g.labels is not None \
            or (sink is not None and _has_emitters(forest)):
        return "dfs", "no level-3 subtree to split (or list/labeled/vertex tasks)"
    if mode == "auto" and kernel_family(g, forest, tasks, sink) != "plan":
        return "dfs", f"{kernel_family(g, forest, tasks, sink)} kernels, not the plan kernel"
    est = frontier_estimate(g, forest, tasks, cfg.bfs_chunk)
    budget = cfg.frontier_bytes or FRONTIER_BUDGET
    if mode == "bfs":
        return "bfs", f"bounded-frontier BFS requested (frontier <= {est} B, blocks of <= {budget} B)"
    avg = g.num_edges / max(g.num_vertices, 1)
    skew = g.max_degree / max(avg, 1e-9)
    if skew < SKEW_FOR_BFS:
        return "dfs", f"degree skew {skew:.1f} < {SKEW_FOR_BFS}: DFS is balanced"
    if est > budget:
        return "dfs", f"level-3 frontier <= {est} B exceeds the {budget} B budget"
    return "bfs", f"level-3 frontier <= {est} B fits the {budget} B budget; degree skew {skew:.1f}"


def _has_emitters(forest: PlanForest) -> bool:
    return any(a == EMIT_MATCH for r in forest.roots for n in iter_nodes(r)
               for a, _ in n.actions.values())


def execute(g: Graph, forest: PlanForest, tasks, sink=None, device: int | None = None,
            rr=None, index=None, flatten: bool = True, run_config: N.RunConfig | None = None,
            instrument: bool = False, lgs: bool = True, search: str = "dfs",
            cfg: ExecutionConfig | None = None, source_split: tuple | None = None):
    """Run one forest on one GPU. Returns (counts, RunStats, stopped, compile).
    ``source_split`` = (split, chunk) overrides how the source-partitioned
    kernels split a round-robin part ``rr`` (source_spec)."""
    dev = N.default_device() if device is None else device
    N.require_device(dev)
    dg = g.device_graph(dev)
    labeled = g.labels is not None
    k = 0 if (instrument or not lgs) else _lgs_clique_k(g, forest, tasks, sink, index)
    if k:
        # bitmap local-graph kernels; the generated plan kernel handles the
        # few sources whose out-degree exceeds the bitmap tiers
        cp = compile_forest(forest, False, False, dg.max_degree, flatten=flatten)
        spec = source_spec(rr, *(source_split or ()))
        words = np.zeros(2, dtype=np.uint64)
        stats = N.RunStats()
        cfg = run_config if run_config is not None else N.RunConfig()
        N.check(N.lib().g2m_clique_count(dg.handle, k, C.byref(spec), cp.handle, C.byref(cfg),
                                         N.ptr(words, C.c_uint64), C.byref(stats)), "clique")
        pid = forest.pattern_ids[0]
        return {pid: int(words[0]) | (int(words[1]) << 64)}, stats, False, cp
    if lgs and not instrument and _is_cycle4_count(g, forest, tasks, sink, index):
        spec = source_spec(rr, *(source_split or ()), family="cycle4")
        words = np.zeros(2, dtype=np.uint64)
        stats = N.RunStats()
        cfg = run_config if run_config is not None else N.RunConfig()
        N.check(N.lib().g2m_cycle4_count(dg.handle, C.byref(spec), C.byref(cfg),
                                         N.ptr(words, C.c_uint64), C.byref(stats)), "cycle4")
        pid = forest.pattern_ids[0]
        return {pid: int(words[0]) | (int(words[1]) << 64)}, stats, False, None
    if lgs and not instrument and _is_diamond_count(g, forest, tasks, sink, index, rr):
        words = np.zeros(2, dtype=np.uint64)
        stats = N.RunStats()
        cfg = run_config if run_config is not None else N.RunConfig()
        rc = N.lib().g2m_diamond_count(dg.handle, C.byref(cfg), N.ptr(words, C.c_uint64),
                                       C.byref(stats))
        if rc == N.G2M_OK:
            pid = forest.pattern_ids[0]
            return {pid: int(words[0]) | (int(words[1]) << 64)}, stats, False, None
        if rc != N.G2M_EUSAGE:          # out-degree beyond the tiers: generated kernel below
            N.check(rc, "diamond")
    if search != "dfs" and not instrument and index is None:
        ecfg = cfg or ExecutionConfig()
        if search == "bfs" or ecfg.search != search:
            ecfg = ExecutionConfig(**{**ecfg.__dict__, "search": search})
        if choose_search(g, forest, tasks, ecfg, sink)[0] == "bfs":
            ce = compile_forest(forest, labeled, False, dg.max_degree, flatten=flatten,
                                frontier="expand")
            cc = compile_forest(forest, labeled, False, dg.max_degree, flatten=flatten,
                                frontier="consume")
            spec, keep = task_spec(tasks, rr=rr)
            words = np.zeros(2 * max(ce.gen.num_patterns, 1), dtype=np.uint64)
            stats = N.RunStats()
            rcfg = run_config if run_config is not None else N.RunConfig()
            # frontier buffer: the whole estimated frontier when it fits the budget
            fbytes = min(frontier_estimate(g, forest, tasks, ecfg.bfs_chunk) + (1 << 20),
                         int(ecfg.frontier_bytes or FRONTIER_BUDGET))
            N.check(N.lib().g2m_run_bfs(ce.handle, cc.handle, dg.handle, C.byref(spec), C.byref(rcfg),
                                        int(ecfg.bfs_chunk), int(fbytes),
                                        N.ptr(words, C.c_uint64), C.byref(stats)), "bfs")
            del keep
            return _counts_from(words, ce.gen.pattern_ids), stats, False, ce
    if (lgs and not instrument and index is None and sink is None
            and forest.parallel_granularity == VERTEX_PARALLEL and isinstance(tasks, VertexTasks)
            and _skewed(g)):
        # a vertex task of a hub is one warp's serial work: run the same plans
        # edge-parallel over the implicit edge list instead (the reference's
        # own vertex/edge agreement, test_executor.py:54-59)
        forest = _edge_form(forest)
        tasks = _default_tasks(g, forest)
    list_mode = sink is not None and _has_emitters(forest)
    cp = compile_forest(forest, labeled, list_mode, dg.max_degree, flatten=flatten,
                        instrument=instrument)
    return _run_kernel(cp, dg, forest, tasks, sink, list_mode, rr=rr, index=index,
                       run_config=run_config)


def _run_kernel(cp: "CompiledPlan", dg, forest: PlanForest, tasks, sink, list_mode: bool,
                rr=None, index=None, run_config: N.RunConfig | None = None):
    """g2m_run (count) or g2m_list (matches to ``sink`` in the reference's
    order) of a compiled kernel; returns (counts, RunStats, stopped, cp)."""
    spec, keep = task_spec(tasks, rr=rr, index=index)
    words = np.zeros(2 * max(cp.gen.num_patterns, 1), dtype=np.uint64)
    stats = N.RunStats()
    cfg = run_config if run_config is not None else N.RunConfig()
    stopped = False
    if not list_mode:
        N.check(N.lib().g2m_run(cp.handle, dg.handle, C.byref(spec), C.byref(cfg),
                                N.ptr(words, C.c_uint64), C.byref(stats)), "run")
    else:
        pids = cp.gen.pattern_ids
        depth = {pid: forest.plans[pid].depth for pid in pids}
        err: list[BaseException] = []

        def on_match(_user, pid, k, n, tuples):
            try:
                name = pids[pid]
                d = depth[name]
                for i in range(int(n)):
                    base = i * k
                    match = tuple(int(tuples[base + j]) for j in range(d))
                    if sink(name, match):
                        return 1
                return 0
            except BaseException as exc:  # surface after the native call returns
                err.append(exc)
                return 1

        cb = N.MATCH_CB(on_match)
        rc = N.lib().g2m_list(cp.handle, dg.handle, C.byref(spec), C.byref(cfg), cb, None,
                              N.ptr(words, C.c_uint64), C.byref(stats))
        if err:
            raise err[0]
        stopped = N.check(rc, "list") == N.G2M_STOPPED
    del keep
    return _counts_from(words, cp.gen.pattern_ids), stats, stopped, cp


def compile_lgs(plan: SearchPlan, list_mode: bool, max_degree: int) -> CompiledPlan:
    """Generate + NVRTC-compile the bitmap local-graph-search kernel of a
    hub-rooted plan (codegen_lgs; cached by generated source)."""
    gen = codegen_lgs.generate_lgs(plan, list_mode=list_mode, max_degree=max_degree)
    return _compile_gen(gen, instrument=False)


# ---------------------------------------------------------------------------
# run_dfs / run_dfs_lgs
# ---------------------------------------------------------------------------

def _default_tasks(g: Graph, forest: PlanForest):
    if forest.parallel_granularity == EDGE_PARALLEL:
        plans = list(forest.plans.values())
        if len(plans) == 1:
            return build_edge_tasks(g, plans[0])
        reduced = all(pl.constrains_first_edge() for pl in plans)
        return EdgeTaskList.implicit(g, reduced=reduced and not g.oriented)
    return VertexTasks(g.num_vertices)


def run_dfs(g: Graph, forest, tasks=None, cfg: ExecutionConfig | None = None,
            sink=None, device: int | None = None) -> RunResult:
    """Run a plan or fused forest to completion on one GPU; exact per-pattern
    counts (executor.py:339-408)."""
    forest = as_forest(forest)
    cfg = cfg or ExecutionConfig()
    if forest.uses_orientation != g.oriented:
        raise ValueError("plan orientation does not match the graph "
                         f"(plan={forest.uses_orientation}, graph={g.oriented})")
    if tasks is None:
        tasks = _default_tasks(g, forest)
    edge_mode = isinstance(tasks, EdgeTaskList)
    if edge_mode and forest.parallel_granularity != EDGE_PARALLEL:
        raise ValueError("edge tasks supplied to a vertex-parallel forest")
    if not edge_mode and forest.parallel_granularity != VERTEX_PARALLEL:
        raise ValueError("vertex tasks supplied to an edge-parallel forest")
    num_tasks = len(tasks)
    workers = resolve_worker_count(cfg, forest.num_buffers, g.max_degree, num_tasks)
    t0 = time.perf_counter()
    counts, st, stopped, _ = execute(g, forest, tasks, sink=sink, device=device,
                                     search=cfg.search, cfg=cfg)
    for pid in forest.pattern_ids:
        counts.setdefault(pid, 0)
    high = tuple(int(st.high_water[i]) if i < 8 else 0 for i in range(forest.num_buffers))
    stats = ExecStats(workers=workers, tasks=num_tasks, num_buffers=forest.num_buffers,
                      buffer_high_water=high, elapsed_s=time.perf_counter() - t0,
                      kernel_ms=float(st.kernel_ms),
                      device=N.default_device() if device is None else device,
                      gpu_warps=int(st.warps))
    return RunResult(counts=counts, stats=stats, stopped_early=stopped)


def run_dfs_lgs(g: Graph, plan: SearchPlan, tasks=None,
                cfg: ExecutionConfig | None = None, sink=None,
                device: int | None = None) -> RunResult:
    """Hub-rooted plans confined to per-task local graphs (executor.py:526-599).
    Preconditions and errors are the reference's; counts equal run_dfs."""
    cfg = cfg or ExecutionConfig()
    p = plan.pattern
    k = p.size
    if p.degree(plan.matching_order.order[0]) != k - 1:
        raise ValueError("local graph search requires a hub-rooted plan")
    if plan.uses_orientation != g.oriented:
        raise ValueError("plan orientation does not match the graph")
    if any(lv.expr.label is not None for lv in plan.levels):
        raise ValueError("local graph search does not support label filters")
    if plan.parallel_granularity == EDGE_PARALLEL:
        if p.degree(plan.matching_order.order[1]) != k - 1:
            raise ValueError("edge-parallel local graph search needs hubs at "
                             "levels 1 and 2; use vertex granularity instead")
        if tasks is None:
            tasks = build_edge_tasks(g, plan)
        anchored = 2
    else:
        if tasks is None:
            tasks = VertexTasks(g.num_vertices)
        anchored = 1
    if anchored + 1 > plan.depth:
        raise ValueError("plan too shallow for local graph search")
    codegen_lgs.check_plan(plan)
    num_tasks = len(tasks)
    workers = resolve_worker_count(cfg, plan.num_buffers, g.max_degree, num_tasks)
    t0 = time.perf_counter()
    forest = as_forest(plan)
    if _lgs_clique_k(g, forest, tasks, sink, None) and not LGS_GENERATED_CLIQUES:
        # k-clique counts: the hand-written bitmap LGS tiers (g2m_clique_count)
        counts, st, stopped, _ = execute(g, forest, tasks, sink=sink, device=device)
    else:
        # every other hub-rooted plan: the generated bitmap LGS kernel
        dev = N.default_device() if device is None else device
        N.require_device(dev)
        dg = g.device_graph(dev)
        list_mode = sink is not None and _has_emitters(forest)
        cp = compile_lgs(plan, list_mode, dg.max_degree)
        counts, st, stopped, _ = _run_kernel(cp, dg, forest, tasks, sink, list_mode)
    counts = {plan.pattern_id: counts.get(plan.pattern_id, 0)}
    high = tuple(int(st.high_water[i]) if i < 8 else 0 for i in range(plan.num_buffers))
    stats = ExecStats(workers=workers, tasks=num_tasks, num_buffers=plan.num_buffers,
                      buffer_high_water=high, elapsed_s=time.perf_counter() - t0,
                      kernel_ms=float(st.kernel_ms),
                      device=N.default_device() if device is None else device,
                      gpu_warps=int(st.warps))
    return RunResult(counts=counts, stats=stats, stopped_early=stopped)


def describe_kernel(forest, labeled: bool = False, list_mode: bool = False,
                    max_degree: int = 1024) -> str:
    """The CUDA source generated for a forest (debug aid, like emit_source)."""
    f = as_forest(forest)
    cap = _slot_capacity(f, labeled, max_degree)
    return codegen.generate(f, labeled=labeled, list_mode=list_mode, smem_slot_cap=cap,
                            warps_per_block=WARPS_PER_BLOCK, stage_words=STAGE_WORDS).source


__all__ = ["BudgetError", "ExecutionConfig", "ExecStats", "RunResult", "StopSearch",
           "WorkerContext", "merge_results", "resolve_worker_count", "run_dfs", "choose_search",
           "run_dfs_lgs", "emit_source", "execute", "compile_forest", "VertexTasks"]
