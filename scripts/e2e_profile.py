"""cProfile of one public-API call (GPU box): where the host time goes."""
import cProfile, pstats, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
import paper_2112_09761_b200 as pm

wl = sys.argv[1] if len(sys.argv) > 1 else "cl4"
spec = bench.graph_spec(type("A", (), {"workload": wl, "graph": None, "scale": None, "n": None})())
g0, off, nbr, info = bench.make_graph(spec, 0, pinned=True)
for _ in range(2):
    bench.api_call(wl, pm.Graph(off, nbr))
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
bench.api_call(wl, pm.Graph(off, nbr))
pr.disable()
print(wl, "api ms", round((time.perf_counter() - t) * 1e3, 2))
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
