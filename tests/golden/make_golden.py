"""Generate the golden fixtures from the REFERENCE package (patminer 0.1.0).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/*.json. Everything here is produced by calling the
reference's own public API; the inputs are seeded generators restated in
tests/graphs.py (checked against the reference's generators below).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))          # tests/ (graphs.py)
import graphs as G                              # noqa: E402

import patminer as pm                           # noqa: E402  (the reference)
from patminer import apps, executor, plan as rplan, pattern as rpat  # noqa: E402
from patminer.cli import gen_synthetic         # noqa: E402

REF_DATA = Path("/root/reference/pkg/data")


def ref_graph(edges, n, labels=None):
    return pm.from_edges(np.asarray(edges, dtype=np.int64).reshape(-1, 2), num_vertices=n,
                         labels=labels)


def sha(arr) -> str:
    return hashlib.sha1(np.ascontiguousarray(arr).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
def analysis_fixture():
    pats = {}
    for k in range(2, 9):
        pats[f"clique{k}"] = rpat.generate_clique(k)
    for k in (3, 4, 5):
        for i, p in enumerate(rpat.generate_all_motifs(k)):
            pats[f"motif{k}_{i}"] = p
            pats[f"motif{k}_{i}_edge"] = p.with_induced("edge")
    pats["diamond"] = rpat.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)])
    pats["cycle4"] = rpat.Pattern(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    pats["book"] = rpat.Pattern(5, [(0, 1), (0, 2), (0, 3), (0, 4), (1, 2), (1, 3), (1, 4)])
    pats["path4"] = rpat.Pattern(4, [(0, 1), (1, 2), (2, 3)])
    pats["lab_path"] = rpat.Pattern(3, [(0, 1), (1, 2)], labels=(0, 1, 0))
    pats["lab_tri"] = rpat.Pattern(3, [(0, 1), (0, 2), (1, 2)], labels=(1, 1, 2))
    pats["lab_wedge"] = rpat.Pattern(3, [(0, 1), (0, 2)], labels=(2, 0, 1))
    pats["cycle5"] = rpat.Pattern(5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)])
    pats["house"] = rpat.Pattern(5, [(0, 1), (1, 2), (2, 3), (3, 0), (0, 4), (1, 4)])
    stats_list = [None, rpat.GraphStats(avg_degree=12.0, num_vertices=3000),
                  rpat.GraphStats(avg_degree=30.6, num_vertices=4194304),
                  rpat.GraphStats(avg_degree=2.0, num_vertices=5)]
    out = {}
    for key, p in pats.items():
        rec = {"size": p.size, "edges": [list(e) for e in p.edges],
               "labels": None if p.labels is None else list(p.labels),
               "induced": p.induced, "name": p.name,
               "canonical": repr(p.canonical_form()),
               "auts": sorted(list(a) for a in rpat.automorphisms(p)),
               "orders": [[list(mo.order), [sorted(c) for c in mo.conn], [sorted(a) for a in mo.anti]]
                          for mo in rpat.enumerate_matching_orders(p)],
               "per_stats": []}
        for st in stats_list:
            mo = rpat.select_matching_order(rpat.enumerate_matching_orders(p), st)
            so = rpat.generate_symmetry_order(p, mo)
            props = rpat.detect_properties(p, mo, so)
            r = {"stats": None if st is None else [st.avg_degree, st.num_vertices],
                 "order": list(mo.order), "symmetry": sorted(list(c) for c in so.constraints),
                 "props": [props.is_clique, sorted(props.hub_vertices),
                           None if props.decomposition is None else list(props.decomposition),
                           props.automorphism_count],
                 "describe": rpat.describe_analysis(p, mo, so),
                 "plans": {}}
            for mode in ("count", "list"):
                for gran in ("edge", "vertex"):
                    for oriented in ((False, True) if p.is_clique() else (False,)):
                        pl = rplan.build_plan(p, mo, so, mode, granularity=gran, oriented=oriented)
                        r["plans"][f"{mode}/{gran}/{int(oriented)}"] = rplan.emit_source(rplan.as_forest(pl))
                        if mode == "count":
                            rw = rplan.apply_counting_rewrite(pl, props)
                            r["plans"][f"{mode}/{gran}/{int(oriented)}/rw"] = rplan.emit_source(rplan.as_forest(rw))
            rec["per_stats"].append(r)
        out[key] = rec
    # fused motif forests
    fused = {}
    for k in (3, 4, 5):
        for gran in ("edge", "vertex"):
            for mode in ("count", "list"):
                plans = []
                for p in rpat.generate_all_motifs(k):
                    mo = rpat.select_matching_order(rpat.enumerate_matching_orders(p))
                    so = rpat.generate_symmetry_order(p, mo)
                    pl = rplan.build_plan(p, mo, so, mode, granularity=gran)
                    if mode == "count":
                        pl = rplan.apply_counting_rewrite(pl, rpat.detect_properties(p, mo, so))
                    plans.append(pl)
                fused[f"{k}/{gran}/{mode}"] = rplan.emit_source(rplan.fuse_multi_pattern(plans))
    motif_names = {k: [p.name for p in rpat.generate_all_motifs(k)] for k in (3, 4, 5)}
    return {"patterns": out, "fused": fused, "motif_names": motif_names}


# ---------------------------------------------------------------------------
WORKLOADS = ["tc", "4-clique", "5-clique", "4-cycle", "diamond", "3-motif", "4-motif"]


def run_workload(g, w):
    if w == "tc":
        return {"triangle": pm.triangle_count(g)}
    if w in ("4-clique", "5-clique"):
        return pm.k_clique(g, int(w[0])).counts
    if w == "4-cycle":
        return pm.subgraph_listing(g, G_cycle4(), mode="count").counts
    if w == "diamond":
        return pm.subgraph_listing(g, G_diamond(), mode="count").counts
    if w in ("3-motif", "4-motif"):
        return {p.name: c for p, c in pm.k_motif(g, int(w[0])).items()}
    raise KeyError(w)


def G_cycle4():
    return rpat.Pattern(4, [(0, 1), (1, 2), (2, 3), (3, 0)])


def G_diamond():
    return rpat.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)])


def counts_fixture():
    graphs = {}
    for f in sorted(REF_DATA.glob("*.el")):
        g = pm.load_edgelist(str(f))
        src = np.repeat(np.arange(g.num_vertices), g.degrees)
        e = np.column_stack([src, g.neighbors.astype(np.int64)])
        e = e[e[:, 0] < e[:, 1]]
        graphs[f"data/{f.name}"] = {"n": g.num_vertices, "edges": e.tolist(), "gen": None}
    for (n, p, seed) in [(20, 0.1, 100), (30, 0.2, 101), (40, 0.3, 102), (50, 0.1, 103),
                         (60, 0.2, 104), (70, 0.05, 200), (95, 0.08, 205), (120, 0.1, 212),
                         (150, 0.05, 300), (200, 0.05, 305), (200, 0.1, 17), (100, 0.1, 31)]:
        graphs[f"er/{n}/{p}/{seed}"] = {"gen": ["er", n, p, seed]}
    graphs["rmat/10"] = {"gen": ["rmat", 10, 16, 1]}
    graphs["rmat/11"] = {"gen": ["rmat", 11, 16, 2]}
    graphs["powerlaw/2000"] = {"gen": ["powerlaw", 2000, 4, 3]}
    out = {}
    for key, spec in graphs.items():
        if spec["gen"] is None:
            g = ref_graph(spec["edges"], spec["n"])
        else:
            kind = spec["gen"][0]
            if kind == "er":
                g = G.er_ref(pm, *spec["gen"][1:])
            elif kind == "rmat":
                g = pm.from_edges(G.rmat_edges(*spec["gen"][1:]), num_vertices=1 << spec["gen"][1])
            else:
                e = gen_synthetic("powerlaw", spec["gen"][1], spec["gen"][2], spec["gen"][3])
                assert np.array_equal(e, G.powerlaw_edges(*spec["gen"][1:])), "powerlaw restatement drifted"
                g = pm.from_edges(e, num_vertices=spec["gen"][1])
        rec = {"spec": spec, "n": g.num_vertices, "slots": g.num_edges,
               "csr_sha": sha(g.row_offsets) + sha(g.neighbors), "counts": {}}
        t0 = time.time()
        for w in WORKLOADS:
            if w == "4-motif" and key in ("rmat/11",):
                continue
            if w == "5-clique" and key == "rmat/11":
                continue
            rec["counts"][w] = {k: int(v) for k, v in run_workload(g, w).items()}
        print(f"  {key}: {time.time() - t0:.1f}s", flush=True)
        out[key] = rec
    return out


# ---------------------------------------------------------------------------
def balg_fixture():
    """SURVEY 8(d) instrumentation of the reference executor."""
    state = {"bytes": 0, "in_member": 0}
    ex = executor
    orig = {n: getattr(ex, n) for n in ("intersect", "intersect_count", "difference", "difference_count")}

    def wrap(fn):
        def inner(a, b, bound=None):
            state["bytes"] += 4 * (len(a) + len(b))
            return fn(a, b, bound)
        return inner

    for n, fn in orig.items():
        setattr(ex, n, wrap(fn))
    TR = ex._TreeRunner
    o_term, o_member, o_edge, o_vertex = TR._term, TR._member, TR.run_edge_task, TR.run_vertex_task

    def term(self, j):
        if not state["in_member"]:
            state["bytes"] += 16
        return o_term(self, j)

    def member(self, expr, v):
        state["in_member"] += 1
        try:
            return o_member(self, expr, v)
        finally:
            state["in_member"] -= 1

    def edge(self, s, d):
        state["bytes"] += 8
        return o_edge(self, s, d)

    def vertex(self, v):
        state["bytes"] += 4
        return o_vertex(self, v)

    TR._term, TR._member, TR.run_edge_task, TR.run_vertex_task = term, member, edge, vertex
    code = ex._TreeRunner.exec_node.__code__
    import inspect
    src, first = inspect.getsourcelines(ex._TreeRunner.exec_node)
    line = first + next(i for i, s in enumerate(src) if "v = int(s[idx])" in s)

    def tracer(frame, event, arg):
        if frame.f_code is code:
            def local(fr, ev, a):
                if ev == "line" and fr.f_lineno == line:
                    state["bytes"] += 4
                return local
            return local
        return None

    out = {}
    graphs = {"er/200/0.1/17": G.er_ref(pm, 200, 0.1, 17),
              "rmat/10": pm.from_edges(G.rmat_edges(10, 16, 1), num_vertices=1 << 10)}
    for key, g in graphs.items():
        out[key] = {}
        for w in ["tc", "diamond", "4-cycle", "4-clique", "5-clique", "3-motif"]:
            state["bytes"] = 0
            sys.settrace(tracer)
            try:
                cfg = executor.ExecutionConfig(lgs="off")
                if w == "tc":
                    c = pm.triangle_count(g, cfg=cfg)
                elif w in ("4-clique", "5-clique"):
                    c = pm.k_clique(g, int(w[0]), cfg=cfg).counts
                elif w == "4-cycle":
                    c = pm.subgraph_listing(g, G_cycle4(), mode="count", cfg=cfg).counts
                elif w == "diamond":
                    c = pm.subgraph_listing(g, G_diamond(), mode="count", cfg=cfg).counts
                else:
                    c = {p.name: v for p, v in pm.k_motif(g, 3, cfg=cfg).items()}
            finally:
                sys.settrace(None)
            out[key][w] = state["bytes"]
            print(f"  balg {key} {w}: {state['bytes']}", flush=True)
    for n, fn in orig.items():
        setattr(ex, n, fn)
    TR._term, TR._member, TR.run_edge_task, TR.run_vertex_task = o_term, o_member, o_edge, o_vertex
    return out


# ---------------------------------------------------------------------------
def list_fixture():
    """Exact match streams (single worker) for list-mode order parity."""
    out = {}
    graphs = {"er/40/0.25/71": G.er_ref(pm, 40, 0.25, 71), "er/30/0.3/8": G.er_ref(pm, 30, 0.3, 8)}
    pats = {"triangle": rpat.generate_clique(3), "4-clique": rpat.generate_clique(4),
            "diamond": G_diamond(), "4-cycle": G_cycle4(),
            "tailed": rpat.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2)], induced="vertex")}
    for gk, g in graphs.items():
        for pk, p in pats.items():
            for gran in ("edge", "vertex"):
                mo = rpat.select_matching_order(rpat.enumerate_matching_orders(p), rpat.GraphStats.of(g))
                so = rpat.generate_symmetry_order(p, mo)
                pl = rplan.build_plan(p, mo, so, "list", granularity=gran)
                stream = []
                executor.run_dfs(g, pl, sink=lambda pid, m: (stream.append(list(m)), False)[1])
                out[f"{gk}|{pk}|{gran}"] = {"order": list(mo.order), "stream": stream}
    return out


def main():
    t0 = time.time()
    print("analysis ...", flush=True)
    (HERE / "analysis.json").write_text(json.dumps(analysis_fixture(), indent=0, sort_keys=True))
    print("lists ...", flush=True)
    (HERE / "lists.json").write_text(json.dumps(list_fixture(), separators=(",", ":")))
    print("algorithmic bytes ...", flush=True)
    (HERE / "balg.json").write_text(json.dumps(balg_fixture(), indent=1, sort_keys=True))
    print("counts ...", flush=True)
    (HERE / "counts.json").write_text(json.dumps(counts_fixture(), indent=1, sort_keys=True))
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
