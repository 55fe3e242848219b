"""GCSR v1 fixtures written by the REFERENCE's own ``save_csr``
(graph.py:293-305). Build container only:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_gcsr.py

Writes tests/golden/{k4_labeled,er60_oriented,rmat8}.gcsr: a labeled graph
from the reference's bundled data, an oriented DAG (``orient``), and a
plain symmetric graph.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import graphs as G  # noqa: E402

import patminer as pm  # noqa: E402  (the reference)

REF_DATA = Path("/root/reference/pkg/data")

k4 = pm.load_edgelist(str(REF_DATA / "k4.el"), labeled=True, label_path=str(REF_DATA / "k4.el.labels"))
pm.save_csr(k4, str(HERE / "k4_labeled.gcsr"))
e, _ = G.er_edges(60, 0.2, 3)
pm.save_csr(pm.orient(pm.from_edges(e, num_vertices=60)), str(HERE / "er60_oriented.gcsr"))
pm.save_csr(pm.from_edges(G.rmat_edges(8, 16, 1), num_vertices=256), str(HERE / "rmat8.gcsr"))
print("ok")
