"""Benchmark: pattern counting on synthetic graphs on N B200s.

Default workload = BASELINE.json configs[1]: 4-clique counting on RMAT
scale 22, edge factor 16 (Graph500 a=.57 b=c=.19, seed 1; E = 64,153,257
undirected edges after dedup), degree-oriented DAG, 1 GPU. The other
configs are workloads of the same line format:

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload cl4|cl5|tc|c4|diamond|mc3|mc4]
                    [--scale S] [--n N] [--impl b200|reference]

    tc, cl4, cl5   k-clique count, RMAT-22 (configs[1]; TC also configs[4])
    c4, diamond    subgraph listing count, RMAT-24 (configs[2]; 4-cycle also configs[4])
    mc3, mc4       k-motif count, power-law n=200,000 m=4 seed 3 (configs[3])

A step is one complete count pass over the whole (N>1: this rank's share of
the) task list with the (oriented) graph resident in HBM, i.e. what
``run_job`` executes after its host-side decisions (apps.prepare_job).
``value`` = E / step time (undirected input edges per second, whole job;
time = max over ranks of the device step time). ``e2e`` runs the same count
through the public API (``pm.k_clique``, ``pm.subgraph_listing``,
``pm.k_motif``) from pinned host CSR buffers every step: H2D of the CSR,
device orientation, the kernels, D2H of the counts.

``--gpus N`` with N > 1 outside torchrun re-launches this script under
``torch.distributed.run`` with N ranks (one per GPU, NCCL; with
G2M_BENCH_BACKEND=gloo the ranks fold onto the visible GPUs). Each rank mines
its share: edge tasks by chunked round-robin with c = 2 * resident warps,
sources of the bitmap-LGS / wedge kernels by the workload estimator
(executor.source_spec). The line carries every rank's kernel time and the
max/mean imbalance.

``parity`` (every line) checks the step's count at full scale two ways:
the specialised kernels against the generated plan kernel (over every task,
or over the same residue class of rank-space sources), and the plan kernel
against the CPU oracle on a seeded task sample (counts are additive over
tasks, executor.py:84-90).

``--impl reference`` times the CPU oracle (oracle/oracle.c, the restatement
of the reference executor) with all host threads on a bounded task sample.
"""
from __future__ import annotations

import argparse
import gc as pygc
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

# name -> (kind, arg, default graph, description)
WORKLOADS = {
    "tc": ("clique", 3, ("rmat", 22), "triangle count"),
    "cl4": ("clique", 4, ("rmat", 22), "k-clique k=4 count"),
    "cl5": ("clique", 5, ("rmat", 22), "k-clique k=5 count"),
    "c4": ("sl", "4-cycle", ("rmat", 24), "subgraph listing 4-cycle count"),
    "diamond": ("sl", "diamond", ("rmat", 24), "subgraph listing diamond count"),
    "mc3": ("motif", 3, ("powerlaw", 200000), "3-motif count (all connected 3-vertex patterns)"),
    "mc4": ("motif", 4, ("powerlaw", 200000), "4-motif count (all connected 4-vertex patterns)"),
}


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def graph_spec(args):
    dkind, dsize = WORKLOADS[args.workload][2]
    kind = args.graph or dkind
    if kind == "rmat":
        return "rmat", args.scale or (dsize if dkind == "rmat" else 22)
    return "powerlaw", args.n or (dsize if dkind == "powerlaw" else 200000)


def make_graph(spec, device: int, pinned: bool, host: bool = False):
    """Seeded edges -> CSR built on the GPU -> host copy (pinned); with
    ``host`` (the CPU reference arm) the CSR is built by numpy instead."""
    import graphs as G
    from paper_2112_09761_b200 import graph as GR
    t0 = time.perf_counter()
    kind, size = spec
    if kind == "rmat" and size >= 25 and not host:
        # too large for the host generator: R-MAT generated on the device
        # (same process, device RNG); the e2e leg's host CSR is its pinned
        # download (the GCSR a user would load)
        g = GR.rmat_device(size, 16, 1, device=device)
        info = {"gen_s": 0.0, "build_s": round(time.perf_counter() - t0, 2),
                "generator": "device R-MAT (counter-based RNG)"}
        if not pinned:
            return g, None, None, info
        import torch
        po = torch.empty(g.num_vertices + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        pn = torch.empty(g.num_edges, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        g.device_graph(device).download_into(po, pn)
        return g, po, pn, info
    if kind == "rmat":
        edges, nv = G.rmat_edges(size, 16, 1), 1 << size
    else:
        edges, nv = G.powerlaw_edges(size, 4, 3), size
    t1 = time.perf_counter()
    if host:
        g = GR.from_edges(edges, num_vertices=nv)
        return g, None, None, {"gen_s": round(t1 - t0, 2), "build_s": round(time.perf_counter() - t1, 2)}
    g = GR.from_edges_device(edges, num_vertices=nv, device=device)
    del edges
    off, nbr = g.row_offsets, g.neighbors     # downloads once
    if pinned:
        import torch
        po = torch.empty(len(off), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        pn = torch.empty(len(nbr), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        po[:] = off
        pn[:] = nbr
        off, nbr = po, pn
    return g, off, nbr, {"gen_s": round(t1 - t0, 2), "build_s": round(time.perf_counter() - t1, 2)}


def patterns_for(workload: str):
    from paper_2112_09761_b200 import pattern as P
    kind, arg, _, _ = WORKLOADS[workload]
    if kind == "clique":
        return [P.generate_clique(arg)]
    if kind == "sl":
        if arg == "4-cycle":
            return [P.Pattern(4, [(0, 1), (1, 2), (2, 3), (3, 0)])]
        return [P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)])]
    return P.generate_all_motifs(arg)


def prepare(workload: str, g):
    """run_job's host-side decisions for this workload (apps.prepare_job):
    orientation, plans, counting rewrite, fusion, task list."""
    from paper_2112_09761_b200 import apps
    kind, arg, _, _ = WORKLOADS[workload]
    job = apps.MiningJob(graph=g, patterns=patterns_for(workload), mode="count")
    if kind == "motif":     # k_motif's granularity rule (apps.py:299-311)
        job.granularity = apps.VERTEX_PARALLEL if arg == 3 else apps.EDGE_PARALLEL
    return apps.prepare_job(job)


def api_call(workload, g):
    import paper_2112_09761_b200 as pm
    kind, arg, _, _ = WORKLOADS[workload]
    if kind == "clique":
        if arg == 3:
            return {"triangle": pm.triangle_count(g)}
        return pm.k_clique(g, arg).counts
    if kind == "sl":
        return pm.subgraph_listing(g, patterns_for(workload)[0], mode="count").counts
    return {p.name: c for p, c in pm.k_motif(g, arg).items()}


def sample_tasks(gd, tasks, m: int, seed: int):
    """A seeded uniform sample of m tasks of the (implicit) task list:
    (positions in the list or None, the tasks as the oracle takes them,
    edge?, list length). A reduced edge list (dst < src slots) is sampled by
    rejection over all slots, so no pass over the whole list is needed; its
    sample then runs on the GPU as an explicit task list."""
    from paper_2112_09761_b200.graph import EdgeTaskList
    off = np.asarray(gd.row_offsets, dtype=np.int64)
    nbr = gd.neighbors
    edge = isinstance(tasks, EdgeTaskList)
    rng = np.random.default_rng(seed)
    if not edge:
        total = gd.num_vertices
        pick = np.sort(rng.choice(total, size=min(m, total), replace=False)).astype(np.int64)
        return pick, pick, False, total
    total = len(tasks)
    slots_all = int(off[-1])
    if tasks.reduced:
        if m >= total:      # small graph: the whole reduced list
            s = np.arange(slots_all, dtype=np.int64)
        else:
            s = np.unique(rng.integers(0, slots_all, size=int(m * 2.5) + 64, dtype=np.int64))
        src = np.searchsorted(off, s, side="right") - 1
        keep = nbr[s].astype(np.int64) < src
        s, src = s[keep][:m], src[keep][:m]
        return None, np.column_stack([src, nbr[s].astype(np.int64)]), True, total
    pick = np.sort(rng.choice(total, size=min(m, total), replace=False)).astype(np.int64)
    src = np.searchsorted(off, pick, side="right") - 1
    return pick, np.column_stack([src, nbr[pick].astype(np.int64)]), True, total


def cpu_sample_run(gd, forest, tasks, target_s: float, threads: int, seed: int = 7):
    """Oracle on a seeded uniform sample of the task list; returns
    (seconds, sampled tasks, total tasks, counts, sample positions, tasks)."""
    from oracle import oracle as O
    m = 2000
    while True:
        pick, tk, edge, total = sample_tasks(gd, tasks, m, seed)
        t0 = time.perf_counter()
        counts, _ = O.run(gd, forest, tasks=tk, edge=edge, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= target_s * 0.5 or m >= total:
            return dt, len(tk), total, counts, pick, tk
        m = int(min(total, m * max(2.0, 0.8 * target_s / max(dt, 1e-3))))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args_n: int) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks on this node and pass rank 0's line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args_n}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    log("relaunching under torchrun:", " ".join(cmd[2:6]), "...")
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# roofline: the specialised kernels' own algorithmic bytes
# ---------------------------------------------------------------------------

def kernel_operands(family: str, gd, forest, tasks, local, rank, args):
    """(operand bytes per step, how, units) of the kernels the step runs.
    lgs / cycle4 / diamond: the specialised algorithm's compulsory operand
    reads (g2m_kernel_work); plan: the instrumented plan kernel's SURVEY
    8(d) bytes (its algorithm is the reference plan)."""
    from paper_2112_09761_b200 import executor as EX
    from paper_2112_09761_b200 import graph as GR
    if family == "lgs":
        ob, probes, bits, src = gd.device_graph(local).kernel_work(0)
        return ob, ("bitmap LGS in rank space: per source u its offsets + N+(u); per member v outside "
                    "the hub core its offsets + N+(v) (local-graph probes); per member in the core one "
                    "4-byte core word per later member (bit tests)"), \
            {"probed_ids": probes, "core_bit_tests": bits, "sources": src}
    if family == "cycle4":
        ob, wedges, upd, src = gd.device_graph(local).kernel_work(1)
        return ob + 8 * upd, ("wedge aggregation: per top vertex r its offsets + N<(r), per v its "
                              "offsets + the wedge ends N(v) & [lo_x, r) (4 B each), plus one 4 B "
                              "counter read-modify-write per wedge (8 B)"), \
            {"wedges": wedges, "sources": src}
    if family in ("diamond", "diamond-allreduce"):
        og = GR.orient(gd, device=local)
        ob, probes, _, src = og.device_graph(local).kernel_work(2)     # support tiers: no hub core
        # + one support counter RMW per triangle edge (3 per triangle found) and
        # the final pass over the support array
        return ob + 8 * og.num_edges, ("edge triangle support on the degree-oriented DAG: the "
                                       "bitmap-LGS operand bytes + a support counter per DAG edge "
                                       "(read+write)"), {"probed_ids": probes, "sources": src}
    return None, None, None


def binding_from_profiles(workload: str, graph: str):
    """ncu evidence (profiles/ncu_summary.json, written from a committed
    `ncu --set full` capture): per-step DRAM bytes and the dominant kernel's
    utilisation of the resources that bind it."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    return json.loads(f.read_text()).get(f"{workload}@{graph}")


# ---------------------------------------------------------------------------
# parity at full scale
# ---------------------------------------------------------------------------

def residue_parity(family, gd, forest, local, counts, P: int, i: int):
    """Specialised kernels vs the generated plan kernel on the same source
    set: the rank-space sources r = i (mod P). Both sides work on the rank
    relabelling (relabelling it again is the identity), the plan kernel over
    the edge tasks whose first vertex is such an r (the reference plans bind
    the clique's DAG source / the 4-cycle's largest vertex at v1)."""
    from paper_2112_09761_b200 import executor as EX
    from paper_2112_09761_b200 import graph as GR
    pid = forest.pattern_ids[0]
    spec_c, _, _, _ = EX.execute(gd, forest, EX._default_tasks(gd, forest), device=local,
                                 rr=(1, P, i), source_split=("rr", 1))
    rg = GR.rank_relabel(gd, device=local)
    off = np.asarray(rg.row_offsets, dtype=np.int64)
    rows = np.arange(i, rg.num_vertices, P, dtype=np.int64)
    if family == "lgs":
        b, e = off[rows], off[rows + 1]
        lens = e - b
        idx = np.repeat(b - np.cumsum(np.concatenate([[0], lens[:-1]])), lens) + np.arange(lens.sum())
        tasks = EX._default_tasks(rg, forest)
        plan_c, _, _, _ = EX.execute(rg, forest, tasks, device=local, index=idx.astype(np.int64),
                                     lgs=False)
    else:   # 4-cycle: reduced edge tasks (r, w), w < r
        from paper_2112_09761_b200.graph import EdgeTaskList
        nbr = rg.neighbors
        pairs = []
        for r in rows:
            seg = nbr[off[r]:off[r + 1]]
            seg = seg[seg < r]
            if len(seg):
                pairs.append(np.column_stack([np.full(len(seg), r, dtype=np.int64),
                                              seg.astype(np.int64)]))
        pairs = np.concatenate(pairs) if pairs else np.empty((0, 2), dtype=np.int64)
        plan_c, _, _, _ = EX.execute(rg, forest, EdgeTaskList(pairs, reduced=True), device=local,
                                     lgs=False)
    del rg
    return {"check": f"specialised kernels vs generated plan kernel on rank-space sources "
                     f"r = {i} (mod {P})",
            "specialised": int(spec_c[pid]), "plan_kernel": int(plan_c[pid]),
            "equal": int(spec_c[pid]) == int(plan_c[pid])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cl4", choices=list(WORKLOADS))
    ap.add_argument("--graph", choices=["rmat", "powerlaw"], default=None)
    ap.add_argument("--scale", type=int, default=None, help="RMAT scale")
    ap.add_argument("--n", type=int, default=None, help="power-law vertices")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--balg-sample", type=float, default=None,
                    help="fraction of tasks for the reference-equivalent bytes (default: all; "
                         "1e-3 for 4-cycle)")
    ap.add_argument("--residue", type=int, default=None,
                    help="P of the residue-class parity check (default per workload)")
    ap.add_argument("--simulate-parts", type=int, default=0,
                    help="1 GPU: run each of P parts of the multi-GPU split in turn and report "
                         "per-part kernel time and max/mean imbalance")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}))
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # G2M_BENCH_BACKEND=gloo: CPU collectives and ranks folded onto the visible
    # GPUs -- exercises the N>1 path on a single-GPU box (timings meaningless)
    backend = os.environ.get("G2M_BENCH_BACKEND", "nccl")
    coll_dev = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "gloo":
            local = local % max(torch.cuda.device_count(), 1)
            coll_dev = "cpu"
        else:
            coll_dev = f"cuda:{local}"
        torch.cuda.set_device(local)
        dist.init_process_group(backend)
    if args.impl == "reference" and rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    kind, warg, _, desc = WORKLOADS[args.workload]
    os.environ["G2M_DEVICE"] = str(local)
    import paper_2112_09761_b200 as pm
    from paper_2112_09761_b200 import distributed as D
    from paper_2112_09761_b200 import executor as EX

    spec = graph_spec(args)
    ref = args.impl == "reference"
    g, off_h, nbr_h, build_info = make_graph(spec, local, pinned=not ref, host=ref)
    E = g.num_edges // 2
    log("graph", spec, build_info, "E", E, "maxdeg", g.max_degree)
    t_prep = time.perf_counter()
    if ref and kind == "clique":       # CPU arm: host orientation, no device work at all
        from util import orient_host
        g = orient_host(g)
    pj = prepare(args.workload, g)
    gd, forest, tasks = pj.graph, pj.forest, pj.tasks
    build_info["prepare_s"] = round(time.perf_counter() - t_prep, 2)   # incl. device orientation
    gname = (f"RMAT-{spec[1]} (ef16, Graph500 a=.57 b=c=.19, seed 1"
             + (", device RNG)" if build_info.get("generator") else ")") if spec[0] == "rmat"
             else f"power-law n={spec[1]} m=4 seed 3 (cli.gen_synthetic)")
    graph_key = f"{spec[0]}{spec[1]}"
    config = {"workload": f"{desc} on {gname}", "patterns": list(forest.pattern_ids),
              "graph": graph_key, "num_vertices": g.num_vertices,
              "undirected_edges": E, "oriented": gd.oriented, "max_degree_task_graph": gd.max_degree,
              "granularity": pj.granularity, "tasks": len(tasks),
              "search": next((d.render() for d in pj.log if d.name == "bounded-bfs"), "dfs"),
              "parallelism": "1 GPU",
              "l2": "inputs larger than L2 (CSR > 126 MB); no flush needed" if gd.num_edges * 4 > 126e6
              else "graph fits L2: measured warm (no flush)"}
    metric = "edges/s"
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        steps = []
        for i in range(args.warmup + args.steps):
            dt, m, total, _, _, _ = cpu_sample_run(gd, forest, tasks, args.cpu_seconds / 4, threads,
                                                seed=100 + i)
            if i >= args.warmup:
                steps.append(dt * total / m)
        t = float(np.mean(steps))
        v = E / t
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "edges/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t * 1000.0, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32 ids / u64 counts", "data": "synthetic",
                "config": config,
                "cpu_baseline": {"value": v, "unit": "edges/s", "cores": threads, "kind": "port",
                                 "cpu_model": cpu_model(),
                                 "sample": f"seeded uniform task sample per step (~{args.cpu_seconds / 4:.0f}s), "
                                           f"extrapolated to all {total} tasks"},
                "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    # ------------------------------------------------------------------ b200
    rr = D.shard(rank, world, device=local)
    family = EX.kernel_family(gd, forest, tasks, rr=rr)
    # diamonds on N > 1 GPUs: the support kernels on each rank's sources, one
    # all-reduce of the support array, C(t, 2) over each rank's slot share
    support_ar = world > 1 and EX._is_diamond_count(gd, forest, tasks, None, None, None)
    if support_ar:
        family = "diamond-allreduce"
    if world > 1:
        config["parallelism"] = (
            f"{world} GPU(s): graph replicated, edge tasks by chunked round-robin (c = 2 x resident warps), "
            f"LGS/wedge sources by the workload estimator "
            f"({EX.SOURCE_SPLIT}:{EX.SOURCE_CHUNK.get(family, '-')})"
            + ("; diamond support summed by one all-reduce of the per-edge support array" if support_ar else ""))

    def run_share(gg, ff, tt):
        if support_ar:
            return D.diamond_count(gg, rank, world, device=local, rr=rr, name=ff.single().pattern.name)
        counts, st, _, _ = EX.execute(gg, ff, tt, device=local, rr=rr, search="auto")
        return counts, st

    def step():   # run_job's search choice (DFS / bounded-frontier BFS), logged as "bounded-bfs"
        return run_share(gd, forest, tasks)

    for _ in range(args.warmup):
        counts, st = step()
        log("warmup step device_ms", round(st.device_ms, 3), "kernel_ms", round(st.kernel_ms, 3), counts)
    if dist is not None:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dev_ms, kern_ms, launches = [], [], 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        counts, st = step()
        dev_ms.append(st.device_ms)
        kern_ms.append(st.kernel_ms)
        launches += int(st.launches)
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    my_ms = float(np.mean(dev_ms))
    my_kms = float(np.mean(kern_ms))
    total_counts = counts
    per_rank = [{"rank": rank, "device_ms": my_ms, "kernel_ms": my_kms, "tasks": int(st.tasks),
                 "count": int(sum(counts.values()))}]
    if dist is not None:   # the job's time is its slowest rank; counts add up exactly
        ms = D.allreduce_max(my_ms, device=coll_dev)
        total_counts = D.allreduce_counts(counts, device=coll_dev)
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank[0])
        per_rank = gathered
    else:
        ms = my_ms
    value = E / (ms / 1000.0)
    kms_all = [r["kernel_ms"] for r in per_rank]
    balance = {"per_rank": per_rank,
               "imbalance_max_over_mean": (max(kms_all) / (sum(kms_all) / len(kms_all)))
               if sum(kms_all) > 0 else None}

    # e2e through the public API from pinned host buffers (N=1), or the
    # upload/orient/run chain per rank (N>1)
    e2e = None
    if not args.no_e2e and off_h is not None:
        h2d = off_h.nbytes + nbr_h.nbytes
        if world == 1 and g.num_edges > 2_000_000_000:
            # a second resident replica (the e2e upload, its rank copy and
            # workspace) does not fit next to the first at RMAT-27: keep the
            # first on the host (its pinned download is the same CSR) and
            # re-upload it after the e2e leg
            if not g.host_resident:
                g._set_host(off_h, nbr_h)
            for gg in {id(g): g, id(gd): gd}.values():
                gg.drop_device_copies()
        e2e_s = []
        nw = max(2, args.warmup)       # the memory pool settles over the first fresh graphs
        for i in range(nw + args.steps):
            if dist is not None:
                dist.barrier()
            t1 = time.perf_counter()
            hg = pm.Graph(off_h, nbr_h)
            if world == 1:
                api_call(args.workload, hg)
            else:
                pr = prepare(args.workload, hg)
                run_share(pr.graph, pr.forest, pr.tasks)
            dt = time.perf_counter() - t1
            del hg
            # the previous call's graphs (and their device replicas) go before the
            # next timed call, not at some later cyclic-GC pass inside it
            pygc.collect()
            if i >= nw:
                e2e_s.append(dt)
        log("e2e steps ms", [round(x * 1000.0, 1) for x in e2e_s])
        e_ms = float(np.mean(e2e_s)) * 1000.0
        if dist is not None:
            e_ms = D.allreduce_max(e_ms, device=coll_dev)
        e2e = {"value": E / (e_ms / 1000.0), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(16 * len(counts) + 8 * 32), "ms_per_step": e_ms,
               "ms_steps": [round(x * 1000.0, 3) for x in e2e_s],
               "path": "public API (pm.k_clique / triangle_count / subgraph_listing / k_motif) on a "
                       "fresh host Graph" if world == 1 else "prepare_job + execute per rank"}

    pk = peaks()
    hbm = pk.get("hbm_gbs") or 6650.0
    kms = max(kms_all)
    # --- reference-equivalent bytes (SURVEY 8(d) B_alg) from the instrumented
    # plan kernel (untimed); also the full-task plan-kernel count for parity
    balg, balg_how, plan_full = None, None, None
    if not args.no_roofline:
        t_b = time.perf_counter()
        frac = args.balg_sample
        if frac is None and kind == "sl" and warg == "4-cycle" and E > 10 ** 7:
            frac = 1e-3     # the reference 4-cycle plan is quadratic in hub degree: sample it
        if frac is None and kind == "clique" and (warg == 5 or E > 2 * 10 ** 8):
            frac = 1e-2     # 5-clique / RMAT-27: the plan kernel over every task takes minutes
        if frac:
            balg = 0
            if rank == 0:
                ntask = len(tasks)
                rng = np.random.default_rng(11)
                idx = np.sort(rng.choice(ntask, size=max(1, int(ntask * frac)), replace=False))
                _, bst, _, _ = EX.execute(gd, forest, tasks, device=local, index=idx, instrument=True)
                balg = int(int(bst.alg_bytes) * ntask / len(idx))
                balg_how = f"sampled: {len(idx)} of {ntask} tasks (seeded uniform), scaled"
        else:
            pc, bst, _, _ = EX.execute(gd, forest, tasks, device=local, rr=rr, instrument=True)
            balg = int(bst.alg_bytes)
            balg_how = "exact: instrumented plan kernel over every task"
            plan_full = pc
            if dist is not None:
                plan_full = D.allreduce_counts(pc, device=coll_dev)
        if dist is not None:   # whole job: bytes add up over ranks
            balg = D.allreduce_counts({"b": balg}, device=coll_dev)["b"]
        log("reference-equivalent bytes", balg, balg_how, "in", round(time.perf_counter() - t_b, 2), "s")

    roof = None
    if not args.no_roofline:
        ob, ob_how, units = kernel_operands(family, gd, forest, tasks, local, rank, args)
        if ob is None:      # the generated plan kernel: its own algorithm is the reference plan
            ob, ob_how, units = balg, "generated plan kernel = the reference plan: " + str(balg_how), None
        achieved = ob / (kms / 1000.0) / 1e9 if ob else None
        prof = binding_from_profiles(args.workload, graph_key) if world == 1 else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if achieved else None,
                "traffic": prof.get("dram_bytes_per_step") if prof and not prof.get("counters_missing") else None,
                "peak_source": "of measured: MEASURED_PEAKS.json hbm_gbs (copy)" if pk.get("hbm_gbs")
                else "of fallback 6650 (B200_PROFILING.md)",
                "algorithmic_bytes_per_step": ob,
                "algorithmic_bytes_def": ob_how,
                "algorithmic_units": units,
                "kernel": {"lgs": "bitmap local-graph clique tiers (concurrent streams)",
                           "cycle4": "4-cycle wedge-aggregation tiers",
                           "diamond": "edge triangle-support tiers + sum C(t,2)",
                           "diamond-allreduce": "edge triangle-support tiers on each rank's sources, "
                                                "all-reduce of the support array, sum C(t,2) per slot share",
                           "plan": "generated plan kernel (DFS or bounded BFS)"}[family],
                "kernel_ms_per_step": kms,
                "kernel_share": kms / ms if ms else None,
                "binding": prof.get("binding") if prof else None,
                "physical_dram_frac": (prof["dram_bytes_per_step"] / (kms / 1000.0) / 1e9 / hbm)
                if prof and prof.get("dram_bytes_per_step") and not prof.get("counters_missing") else None,
                "ncu_source": prof.get("source") if prof else None,
                "reference_equivalent_bytes_per_step": balg,
                "reference_equivalent_gbs": balg / (kms / 1000.0) / 1e9 if balg else None,
                "reference_equivalent_how": balg_how}

    # --- parity at full scale
    parity = None
    cpu = None
    if not args.no_parity:
        parity = {}
        pid_counts = {k: int(v) for k, v in total_counts.items()}
        if plan_full is not None:
            parity["full_vs_plan_kernel"] = {
                "check": "step count vs the generated plan kernel over every task",
                "plan_kernel": {k: int(v) for k, v in plan_full.items()},
                "equal": {k: int(v) for k, v in plan_full.items()} == pid_counts}
        elif family in ("lgs", "cycle4") and rank == 0 and world == 1:
            P = args.residue or (4001 if family == "cycle4" else 101)
            # the class whose top member is rank nv - P: it skips the P - 1 highest
            # ranks, the hubs whose 4-cycle plan-kernel work is quadratic in degree
            i = (gd.num_vertices % P) if family == "cycle4" else 7 % P
            parity["full_vs_plan_kernel"] = residue_parity(family, gd, forest, local, counts, P, i)
        elif family in ("diamond",) and world == 1:
            pc, _, _, _ = EX.execute(gd, forest, tasks, device=local, lgs=False)
            parity["full_vs_plan_kernel"] = {
                "check": "step count vs the generated plan kernel over every task",
                "plan_kernel": {k: int(v) for k, v in pc.items()},
                "equal": {k: int(v) for k, v in pc.items()} == pid_counts}
        elif family == "plan" and world == 1:
            # the step may run bounded BFS or the edge form of a vertex forest;
            # an explicit index over every task pins plain DFS at the plan's
            # own granularity
            pc, _, _, _ = EX.execute(gd, forest, tasks, device=local,
                                     index=np.arange(len(tasks), dtype=np.int64), lgs=False)
            parity["full_vs_plan_kernel"] = {
                "check": "step count (search chosen by run_job) vs plain DFS of the plan kernel "
                         "over every task at the plan's granularity",
                "plan_kernel": {k: int(v) for k, v in pc.items()},
                "equal": {k: int(v) for k, v in pc.items()} == pid_counts}
    if rank == 0 and world == 1 and not (args.no_cpu_baseline and args.no_parity):
        dt, m, total, ocounts, pick, tk_s = cpu_sample_run(gd, forest, tasks, args.cpu_seconds, threads)
        tcpu = dt * total / m
        if not args.no_cpu_baseline:
            cpu = {"value": E / tcpu, "unit": "edges/s", "cores": threads, "kind": "port",
                   "cpu_model": cpu_model(),
                   "sample": f"{m} of {total} tasks (seeded uniform), {dt:.1f}s, extrapolated"}
        if parity is not None:
            if pick is None:    # reduced edge list: the sampled tasks explicitly
                from paper_2112_09761_b200.graph import EdgeTaskList
                gc, _, _, _ = EX.execute(gd, forest, EdgeTaskList(tk_s, reduced=True), device=local,
                                         lgs=False)
            else:
                gc, _, _, _ = EX.execute(gd, forest, tasks, device=local, index=pick, lgs=False)
            parity["sample_vs_oracle"] = {
                "check": "generated plan kernel vs the CPU oracle on the same seeded task sample",
                "sample_tasks": int(m), "of_tasks": int(total),
                "oracle": {k: int(v) for k, v in ocounts.items()},
                "plan_kernel": {k: int(v) for k, v in gc.items()},
                "equal": {k: int(v) for k, v in gc.items()} == {k: int(v) for k, v in ocounts.items()}}
    if parity is not None:
        oks = [v["equal"] for v in parity.values()]
        parity["all_equal"] = bool(oks) and all(oks)

    # --- multi-GPU split simulated on one GPU: each part in turn
    sim = None
    if args.simulate_parts > 1 and world == 1:
        sim = {}
        P = args.simulate_parts
        splits = ([("est", EX.SOURCE_CHUNK[family]), ("rr", 1)] if family in ("lgs", "cycle4")
                  else [(None, None)])
        if family in ("lgs", "cycle4") and os.environ.get("G2M_SIM_SPLITS"):
            # e.g. "est:1,est:16,rr:1": every listed source split in one process
            splits = [(a, int(b or 1)) for a, _, b in
                      (x.partition(":") for x in os.environ["G2M_SIM_SPLITS"].split(","))]
        for split, chunk in splits:
            part_ms, tot = [], {}
            for i in range(P):
                rr_i = D.shard(i, P, device=local)
                c, st_i, _, _ = EX.execute(gd, forest, tasks, device=local, rr=rr_i, search="auto",
                                           source_split=(split, chunk) if split else None)
                part_ms.append(float(st_i.kernel_ms))
                for k, v in c.items():
                    tot[k] = tot.get(k, 0) + int(v)
            key = f"{split}:{chunk}" if split else "chunked_rr"
            sim[key] = {"parts": P, "kernel_ms": part_ms,
                        "imbalance_max_over_mean": max(part_ms) / (sum(part_ms) / P) if sum(part_ms) else None,
                        "counts_equal_whole": tot == {k: int(v) for k, v in total_counts.items()}}
            log("simulated split", key, sim[key]["imbalance_max_over_mean"])

    line = {"metric": metric, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 ids / u64 counts",
            "data": "synthetic (seeded generators; real datasets unavailable offline)",
            "config": config, "counts": {k: int(v) for k, v in total_counts.items()},
            "kernel_ms_per_step": kms, "wall_s_timed": wall,
            "gpu_launches": launches, "clocks": clocks, "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "balance": balance,
            "partition_sim": sim, "kernel_family": family, "build": build_info}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
