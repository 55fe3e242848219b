"""Golden FSM results from the REFERENCE's own run_bounded_bfs (fsm.py:107-210).
Build container only:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_fsm.py

Writes tests/golden/fsm.json: per case the frequent patterns, all supports,
parent -> child pairs and blocks processed (pattern keys as repr strings).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import graphs as G  # noqa: E402

from patminer import fsm as rfsm  # noqa: E402  (the reference)
from patminer import graph as rgraph  # noqa: E402
from patminer.executor import ExecutionConfig  # noqa: E402

CASES = []
for seed in (4, 5, 6):
    for sigma in (1, 2, 3):
        CASES.append({"gen": ["er", 26, 0.15, seed, 3], "max_edges": 3, "sigma": sigma})
CASES.append({"gen": ["er", 30, 0.15, 41, 3], "max_edges": 3, "sigma": 2})
CASES.append({"gen": ["er", 24, 0.2, 7, 3], "max_edges": 2, "sigma": 1, "block": 8})
CASES.append({"gen": ["er", 40, 0.12, 9, 4], "max_edges": 4, "sigma": 3})
CASES.append({"gen": ["er", 20, 0.3, 11, 2], "max_edges": 4, "sigma": 4, "pruning": False})
CASES.append({"gen": ["tiny"], "max_edges": 1, "sigma": 1})

out = []
for c in CASES:
    if c["gen"][0] == "tiny":
        g = rgraph.from_edges(np.array([(0, 1), (1, 2)]), labels=np.array([0, 0, 1]))
    else:
        _, n, p, seed, nl = c["gen"]
        g = G.er_ref(rgraph, n, p, seed, labels=nl)
    cfg = ExecutionConfig(bfs_block_size=c.get("block", 1 << 20))
    res = rfsm.run_bounded_bfs(g, c["max_edges"], c["sigma"], cfg=cfg, label_pruning=c.get("pruning", True))
    out.append({**c,
                "frequent": {repr(k): v for k, v in res.frequent.items()},
                "all_supports": {repr(k): v for k, v in res.all_supports.items()},
                "parent_child": sorted([repr(a), repr(b)] for a, b in res.parent_child),
                "blocks_processed": res.blocks_processed})
(HERE / "fsm.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")
print(len(out), "cases")
