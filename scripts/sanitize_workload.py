"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the hot path on small seeded graphs, with the
shared-memory variants forced on (two-level window and hash probes, the
TMA-staged pair tier, the 4-cycle staging and grid tiers), each count
checked against the generated plan kernel.

    compute-sanitizer --tool racecheck python scripts/sanitize_workload.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import graphs as G  # noqa: E402
import paper_2112_09761_b200 as pm  # noqa: E402
from paper_2112_09761_b200 import executor as EX  # noqa: E402
from paper_2112_09761_b200 import graph as GR  # noqa: E402
from paper_2112_09761_b200 import pattern as P  # noqa: E402
from paper_2112_09761_b200 import plan as PL  # noqa: E402
from util import cycle4, diamond, make_plan  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 11
g = GR.from_edges(G.rmat_edges(scale, 16, 2), num_vertices=1 << scale)
og = pm.orient(g)
bad = 0


def check(name, got, want):
    global bad
    ok = got == want
    bad += not ok
    print(f"{name}: {'ok' if ok else 'MISMATCH'} {got} {want}", flush=True)


envs = [{}, {"G2M_DIRECT_MAX": "64"}, {"G2M_DIRECT_MAX": "0"}, {"G2M_PAIR_BULK": "1"},
        {"G2M_TIER_STREAMS": "4"}]
for k in (3, 4, 5):
    f = PL.as_forest(make_plan(P.generate_clique(k), g, oriented=True))
    tasks = EX._default_tasks(og, f)
    want = EX.execute(og, f, tasks, lgs=False)[0]
    for e in envs:
        os.environ.update(e)
        og2 = pm.orient(g)
        check(f"clique k={k} {e}", EX.execute(og2, f, EX._default_tasks(og2, f))[0], want)
        for key in e:
            os.environ.pop(key)
for pat, nm in ((cycle4(), "4-cycle"), (diamond(), "diamond")):
    f = PL.as_forest(make_plan(pat, g))
    tasks = EX._default_tasks(g, f)
    want = EX.execute(g, f, tasks, lgs=False)[0]
    for e in ([{}, {"G2M_C4_STAGE_CAP": "2000"}, {"G2M_C4_STAGE_CAP": "0", "G2M_C4_RANGE": "1024"}]
              if nm == "4-cycle" else [{}]):
        os.environ.update(e)
        g2 = GR.from_edges(G.rmat_edges(scale, 16, 2), num_vertices=1 << scale)
        check(f"{nm} {e}", EX.execute(g2, f, EX._default_tasks(g2, f))[0], want)
        for key in e:
            os.environ.pop(key)
m = pm.k_motif(g, 3)
print("3-motif", {p.name: c for p, c in m.items()})
m = pm.k_motif(GR.from_edges(G.rmat_edges(9, 8, 3), num_vertices=1 << 9), 4)
print("4-motif", {p.name: c for p, c in m.items()})
print("MISMATCHES", bad)
sys.exit(1 if bad else 0)
