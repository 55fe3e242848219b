"""A/B of the clique tier launch modes on one graph (one process, graph
built once): G2M_TIER_STREAMS unset (8 side streams), 1 (one stream, no
host syncs), 2..4 side streams; then G2M_DEBUG for per-tier times."""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import graphs as G
import paper_2112_09761_b200 as pm
from paper_2112_09761_b200 import executor as EX
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import apps

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "3,4,5").split(",")]
modes = (sys.argv[3] if len(sys.argv) > 3 else "8,1,2,4").split(",")
g = GR.from_edges_device(G.rmat_edges(scale, 16, 1), num_vertices=1 << scale)
for k in ks:
    pj = apps.prepare_job(apps.MiningJob(graph=g, patterns=[P.generate_clique(k)], mode="count"))
    for m in modes:
        os.environ["G2M_TIER_STREAMS"] = m
        ms = []
        for i in range(6):
            c, st, _, _ = EX.execute(pj.graph, pj.forest, pj.tasks)
            ms.append(st.kernel_ms)
        print(f"k={k} streams={m} kernel_ms {np.round(ms, 2).tolist()} min {min(ms[2:]):.2f} mean {np.mean(ms[2:]):.2f} counts {c}", flush=True)
    os.environ.pop("G2M_TIER_STREAMS")
    os.environ["G2M_DEBUG"] = "1"
    c, st, _, _ = EX.execute(pj.graph, pj.forest, pj.tasks)
    print(f"k={k} serial-debug kernel_ms {st.kernel_ms:.2f}", flush=True)
    os.environ.pop("G2M_DEBUG")
