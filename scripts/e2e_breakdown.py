"""Where the end-to-end time of one public-API call goes (GPU box)."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import bench
import paper_2112_09761_b200 as pm
from paper_2112_09761_b200 import graph as GR, executor as EX, apps

wl = sys.argv[1] if len(sys.argv) > 1 else "cl4"
spec = bench.graph_spec(type("A", (), {"workload": wl, "graph": None, "scale": None, "n": None})())
g0, off, nbr, info = bench.make_graph(spec, 0, pinned=True)
print("graph", spec, info, flush=True)
for rep in range(3):
    T = {}
    t = time.perf_counter(); hg = pm.Graph(off, nbr); T["Graph()"] = time.perf_counter() - t
    t = time.perf_counter(); hg.device_graph(0); T["upload"] = time.perf_counter() - t
    t = time.perf_counter(); pj = bench.prepare(wl, hg); T["prepare_job(orient..)"] = time.perf_counter() - t
    t = time.perf_counter(); c, st, _, _ = EX.execute(pj.graph, pj.forest, pj.tasks, search="auto"); T["execute#1"] = time.perf_counter() - t
    T["  kernel_ms#1"] = st.kernel_ms / 1e3; T["  device_ms#1"] = st.device_ms / 1e3
    t = time.perf_counter(); c, st, _, _ = EX.execute(pj.graph, pj.forest, pj.tasks, search="auto"); T["execute#2"] = time.perf_counter() - t
    t = time.perf_counter(); bench.api_call(wl, pm.Graph(off, nbr)); T["api_call total"] = time.perf_counter() - t
    print(rep, {k: round(v * 1000, 1) for k, v in T.items()}, flush=True)
