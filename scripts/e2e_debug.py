"""Phase times of public-API calls (G2M_DEBUG=1 native phase lines on stderr)."""
import os, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
import paper_2112_09761_b200 as pm

wl = sys.argv[1] if len(sys.argv) > 1 else "cl4"
spec = bench.graph_spec(type("A", (), {"workload": wl, "graph": None, "scale": None, "n": None})())
g0, off, nbr, info = bench.make_graph(spec, 0, pinned=True)
for rep in range(3):
    t = time.perf_counter(); bench.api_call(wl, pm.Graph(off, nbr)); print(rep, "plain api ms", round((time.perf_counter() - t) * 1e3, 2), flush=True)
os.environ["G2M_DEBUG"] = "1"
for rep in range(2):
    t = time.perf_counter(); bench.api_call(wl, pm.Graph(off, nbr)); print(rep, "debug api ms", round((time.perf_counter() - t) * 1e3, 2), flush=True)
