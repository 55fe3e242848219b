"""A/B of environment switches on the clique / 4-cycle / diamond kernels
(one process, graph built once).

    python scripts/ab_env.py <scale> <cl3,cl4,cl5,c4,diamond> "A=1;B=2|A=0|..." [debug]

Each '|'-separated setting is applied (env vars read by libg2m at each call)
and the workload run 6 times; prints kernel_ms per run and the counts. With
'debug', one more G2M_DEBUG run per setting prints per-tier times to stderr."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import graphs as G  # noqa: E402
from paper_2112_09761_b200 import apps  # noqa: E402
from paper_2112_09761_b200 import executor as EX  # noqa: E402
from paper_2112_09761_b200 import graph as GR  # noqa: E402
from paper_2112_09761_b200 import pattern as P  # noqa: E402

scale = int(sys.argv[1])
works = sys.argv[2].split(",")
settings = sys.argv[3].split("|")
debug = len(sys.argv) > 4 and sys.argv[4] == "debug"
g = GR.rmat_device(scale, 16, 1) if scale >= 25 else GR.from_edges_device(G.rmat_edges(scale, 16, 1), num_vertices=1 << scale)
for w in works:
    if w.startswith("cl"):
        pats = [P.generate_clique(int(w[2:]))]
    elif w == "c4":
        pats = [P.Pattern(4, [(0, 1), (1, 2), (2, 3), (3, 0)])]
    else:
        pats = [P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)])]
    pj = apps.prepare_job(apps.MiningJob(graph=g, patterns=pats, mode="count"))
    for s in settings:
        kv = [x.split("=", 1) for x in s.split(";") if "=" in x]
        for k, v in kv:
            os.environ[k] = v
        ms = []
        for i in range(int(os.environ.get("AB_REPS", "6"))):
            c, st, _, _ = EX.execute(pj.graph, pj.forest, pj.tasks)
            ms.append(st.kernel_ms)
        print(f"{w} [{s}] kernel_ms {np.round(ms, 2).tolist()} min {min(ms[1:] or ms):.2f} mean {np.mean(ms[1:] or ms):.2f} counts {c}",
              flush=True)
        if debug:
            os.environ["G2M_DEBUG"] = "1"
            print(f"--- {w} [{s}] debug", file=sys.stderr, flush=True)
            EX.execute(pj.graph, pj.forest, pj.tasks)
            os.environ.pop("G2M_DEBUG")
        for k, _ in kv:
            os.environ.pop(k)
