"""Benchmark: pattern counting on synthetic graphs on N B200s.

Default workload = BASELINE.json configs[1]: 4-clique counting on RMAT
scale 22, edge factor 16 (Graph500 a=.57 b=c=.19, seed 1; E = 64,153,257
undirected edges after dedup), degree-oriented DAG, 1 GPU. The other
configs are workloads of the same line format:

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload cl4|cl5|tc|c4|diamond|mc3|mc4]
                    [--scale S] [--n N] [--impl b200|reference]

    tc, cl4, cl5   k-clique count, RMAT-22 (configs[1]; TC also configs[4])
    c4, diamond    subgraph listing count, RMAT-24 (configs[2])
    mc3, mc4       k-motif count, power-law n=200,000 m=4 seed 3 (configs[3])

A step is one complete count pass over the whole (N>1: this rank's chunked
round-robin share of the) task list with the (oriented) graph resident in
HBM, i.e. what ``run_job`` executes after its host-side decisions
(apps.prepare_job). ``value`` = E / step time (undirected input edges per
second, whole job; time = max over ranks of the device step time). ``e2e``
runs the same count through the public API (``pm.k_clique``,
``pm.subgraph_listing``, ``pm.k_motif``) from pinned host CSR buffers every
step: H2D of the CSR, device orientation, the kernels, D2H of the counts.
``--impl reference`` times the CPU oracle (oracle/oracle.c, the restatement
of the reference executor) with all host threads on a bounded task sample.
"""
from __future__ import annotations

import argparse
import json
import os
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
        # (same process, device RNG); no host copy (no e2e at this scale)
        g = GR.rmat_device(size, 16, 1, device=device)
        return g, None, None, {"gen_s": 0.0, "build_s": round(time.perf_counter() - t0, 2),
                               "generator": "device R-MAT (counter-based RNG)"}
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


def cpu_sample_run(gd, forest, tasks, target_s: float, threads: int, seed: int = 7):
    """Oracle on a seeded uniform sample of the task list; returns
    (seconds, sampled tasks, total tasks, counts)."""
    from oracle import oracle as O
    from paper_2112_09761_b200.graph import EdgeTaskList
    off = np.asarray(gd.row_offsets, dtype=np.int64)
    nbr = gd.neighbors
    edge = isinstance(tasks, EdgeTaskList)
    slots = None
    if edge and tasks.reduced:
        src_all = np.repeat(np.arange(gd.num_vertices, dtype=np.int64), np.diff(off))
        slots = np.flatnonzero(nbr.astype(np.int64) < src_all)
        del src_all
    total = len(slots) if slots is not None else (int(off[-1]) if edge else gd.num_vertices)
    rng = np.random.default_rng(seed)

    def sample(m):
        pick = rng.choice(total, size=min(m, total), replace=False)
        pick.sort()
        if not edge:
            return pick.astype(np.int64)
        s = slots[pick] if slots is not None else pick
        src = np.searchsorted(off, s, side="right") - 1
        return np.column_stack([src, nbr[s].astype(np.int64)])

    m = 2000
    while True:
        tk = sample(m)
        t0 = time.perf_counter()
        counts, _ = O.run(gd, forest, tasks=tk, edge=edge, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= target_s * 0.5 or m >= total:
            return dt, len(tk), total, counts
        m = int(min(total, m * max(2.0, 0.8 * target_s / max(dt, 1e-3))))


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
    ap.add_argument("--balg-sample", type=float, default=None,
                    help="fraction of tasks for the algorithmic-byte count (default: all; 1e-3 for 4-cycle)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
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
    config = {"workload": f"{desc} on {gname}", "patterns": list(forest.pattern_ids),
              "graph": f"{spec[0]}{spec[1]}", "num_vertices": g.num_vertices,
              "undirected_edges": E, "oriented": gd.oriented, "max_degree_task_graph": gd.max_degree,
              "granularity": pj.granularity, "tasks": len(tasks),
              "search": next((d.render() for d in pj.log if d.name == "bounded-bfs"), "dfs"),
              "parallelism": f"{world} GPU(s), chunked round-robin tasks, graph replicated"
              if world > 1 else "1 GPU",
              "l2": "inputs larger than L2 (CSR > 126 MB); no flush needed" if gd.num_edges * 4 > 126e6
              else "graph fits L2: measured warm (no flush)"}
    metric = "edges/s"

    if args.impl == "reference":
        threads = os.cpu_count() or 1
        steps = []
        for i in range(args.warmup + args.steps):
            dt, m, total, _ = cpu_sample_run(gd, forest, tasks, args.cpu_seconds / 4, threads,
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
                                 "sample": f"seeded uniform task sample per step (~{args.cpu_seconds / 4:.0f}s), "
                                           f"extrapolated to all {total} tasks"},
                "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    # ------------------------------------------------------------------ b200
    rr = D.shard(rank, world)

    def step():   # run_job's search choice (DFS / bounded-frontier BFS), logged as "bounded-bfs"
        counts, st, _, _ = EX.execute(gd, forest, tasks, device=local, rr=rr, search="auto")
        return counts, st

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
    total_counts = counts
    if dist is not None:   # the job's time is its slowest rank; counts add up exactly
        ms = D.allreduce_max(my_ms, device=coll_dev)
        total_counts = D.allreduce_counts(counts, device=coll_dev)
    else:
        ms = my_ms
    value = E / (ms / 1000.0)

    # e2e through the public API from pinned host buffers (N=1), or the
    # upload/orient/run chain per rank (N>1)
    e2e = None
    if not args.no_e2e and off_h is not None:
        h2d = off_h.nbytes + nbr_h.nbytes
        e2e_s = []
        nw = max(1, args.warmup // 2)
        for i in range(nw + args.steps):
            if dist is not None:
                dist.barrier()
            t1 = time.perf_counter()
            hg = pm.Graph(off_h, nbr_h)
            if world == 1:
                api_call(args.workload, hg)
            else:
                pr = prepare(args.workload, hg)
                EX.execute(pr.graph, pr.forest, pr.tasks, device=local, rr=rr, search="auto")
            dt = time.perf_counter() - t1
            del hg
            if i >= nw:
                e2e_s.append(dt)
        e_ms = float(np.mean(e2e_s)) * 1000.0
        if dist is not None:
            e_ms = D.allreduce_max(e_ms, device=coll_dev)
        e2e = {"value": E / (e_ms / 1000.0), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(16 * len(counts) + 8 * 32), "ms_per_step": e_ms,
               "path": "public API (pm.k_clique / triangle_count / subgraph_listing / k_motif) on a "
                       "fresh host Graph" if world == 1 else "prepare_job + execute per rank"}

    pk = peaks()
    hbm = pk.get("hbm_gbs") or 6650.0
    kms = float(np.mean(kern_ms))
    # SURVEY 8(d) algorithmic bytes of the reference plan over this rank's
    # tasks, from the instrumented generated kernel (run once, untimed)
    balg, balg_how = None, None
    if not args.no_roofline:
        t_b = time.perf_counter()
        frac = args.balg_sample
        if frac is None and kind == "sl" and WORKLOADS[args.workload][1] == "4-cycle" and E > 10 ** 7:
            frac = 1e-3     # the reference 4-cycle plan is quadratic in hub degree: sample it
        if frac:
            # seeded uniform sample of the whole job's tasks through the
            # instrumented plan kernel, scaled up (rank 0 only)
            balg = 0
            if rank == 0:
                ntask = len(tasks)
                rng = np.random.default_rng(11)
                idx = np.sort(rng.choice(ntask, size=max(1, int(ntask * frac)), replace=False))
                _, bst, _, _ = EX.execute(gd, forest, tasks, device=local, index=idx, instrument=True)
                balg = int(int(bst.alg_bytes) * ntask / len(idx))
                balg_how = f"sampled: {len(idx)} of {ntask} tasks (seeded uniform), scaled"
        else:
            _, bst, _, _ = EX.execute(gd, forest, tasks, device=local, rr=rr, instrument=True)
            balg = int(bst.alg_bytes)
            balg_how = "exact: instrumented plan kernel over every task"
        if dist is not None:   # whole job: bytes add up over ranks, time is the slowest rank's
            balg = D.allreduce_counts({"b": balg}, device=coll_dev)["b"]
            kms = D.allreduce_max(kms, device=coll_dev)
        log("algorithmic bytes", balg, balg_how, "in", round(time.perf_counter() - t_b, 2), "s")
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists() and world == 1:
        traffic = json.loads(tfile.read_text()).get(f"{args.workload}@{config['graph']}")
    achieved = balg / (kms / 1000.0) / 1e9 if balg else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm if achieved else None,
            "traffic": traffic.get("dram_bytes_per_step") if traffic else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if pk.get("hbm_gbs")
            else "fallback 6650 (B200_PROFILING.md)",
            "algorithmic_bytes_per_step": balg,
            "algorithmic_bytes_how": balg_how,
            "algorithmic_bytes_def": "SURVEY 8(d): 4B x (|A|+|B|) per reference set op + 4B per "
                                     "DESCEND candidate + 16B per list opened + 8B/4B per edge/vertex task",
            "kernel": "mining kernels of one step" + (" (bitmap LGS tiers)" if kind == "clique"
                                                      else " (generated plan kernel)"),
            "kernel_ms_per_step": kms,
            "kernel_share": kms / my_ms if my_ms else None,
            "physical_dram_frac": (traffic["dram_bytes_per_step"] / (kms / 1000.0) / 1e9 / hbm)
            if traffic else None,
            "traffic_source": traffic.get("source") if traffic else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        dt, m, total, _ = cpu_sample_run(gd, forest, tasks, args.cpu_seconds, threads)
        tcpu = dt * total / m
        cpu = {"value": E / tcpu, "unit": "edges/s", "cores": threads, "kind": "port",
               "sample": f"{m} of {total} tasks (seeded uniform), {dt:.1f}s, extrapolated"}

    line = {"metric": metric, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 ids / u64 counts",
            "data": "synthetic (seeded generators; real datasets unavailable offline)",
            "config": config, "counts": {k: int(v) for k, v in total_counts.items()},
            "kernel_ms_per_step": kms, "wall_s_timed": wall,
            "gpu_launches": launches, "clocks": clocks, "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "build": build_info}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
