"""The CPU oracle (oracle/oracle.c, a restatement of the reference executor)
is pinned against the reference's own outputs: counts on every golden graph
and workload, the SURVEY 8(d) algorithmic bytes, and exact list streams."""
import json
from pathlib import Path

import numpy as np
import pytest

import graphs as G
from oracle import oracle as O
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import plan as PL
from util import analyze, cycle4, diamond, orient_host

GOLD = Path(__file__).parent / "golden"
COUNTS = json.loads((GOLD / "counts.json").read_text())
BALG = json.loads((GOLD / "balg.json").read_text())
LISTS = json.loads((GOLD / "lists.json").read_text())


def build_graph(key, rec):
    spec = rec["spec"]
    if spec["gen"] is None:
        return GR.from_edges(np.asarray(spec["edges"], dtype=np.int64).reshape(-1, 2),
                             num_vertices=spec["n"])
    kind = spec["gen"][0]
    if kind == "er":
        return G.er(*spec["gen"][1:])
    if kind == "rmat":
        return GR.from_edges(G.rmat_edges(*spec["gen"][1:]), num_vertices=1 << spec["gen"][1])
    return GR.from_edges(G.powerlaw_edges(*spec["gen"][1:]), num_vertices=spec["gen"][1])


def forest_for(workload, g, lgs_off=True):
    """The forest run_job builds for a workload (apps.py:90-239), plus the
    graph it runs on (oriented for cliques)."""
    stats = P.GraphStats.of(g)
    if workload == "tc":
        pats = [P.generate_clique(3)]
    elif workload in ("4-clique", "5-clique"):
        pats = [P.generate_clique(int(workload[0]))]
    elif workload == "4-cycle":
        pats = [cycle4()]
    elif workload == "diamond":
        pats = [diamond()]
    else:
        pats = P.generate_all_motifs(int(workload[0]))
    cliques = all(p.is_clique() for p in pats)
    gran = "vertex" if workload == "3-motif" else "edge"
    plans = []
    for p in pats:
        mo = P.select_matching_order(P.enumerate_matching_orders(p), stats)
        so = P.generate_symmetry_order(p, mo)
        pl = PL.build_plan(p, mo, so, "count", granularity=gran, oriented=cliques)
        pl = PL.apply_counting_rewrite(pl, P.detect_properties(p, mo, so))
        plans.append(pl)
    return PL.fuse_multi_pattern(plans), (orient_host(g) if cliques else g)


_graph_cache = {}


def graph(key):
    if key not in _graph_cache:
        _graph_cache[key] = build_graph(key, COUNTS[key])
    return _graph_cache[key]


CASES = [(k, w) for k in sorted(COUNTS) for w in sorted(COUNTS[k]["counts"])]


@pytest.mark.parametrize("key,workload", CASES)
def test_oracle_counts_match_reference(key, workload):
    g = graph(key)
    assert g.num_vertices == COUNTS[key]["n"] and g.num_edges == COUNTS[key]["slots"]
    forest, gg = forest_for(workload, g)
    got, _ = O.run(gg, forest, threads=4)
    assert got == COUNTS[key]["counts"][workload]


def test_generators_reproduce_reference_csr():
    import hashlib
    for key in COUNTS:
        g = graph(key)
        h = hashlib.sha1(np.ascontiguousarray(g.row_offsets).tobytes()).hexdigest() + \
            hashlib.sha1(np.ascontiguousarray(g.neighbors).tobytes()).hexdigest()
        assert h == COUNTS[key]["csr_sha"], key


@pytest.mark.parametrize("key", sorted(BALG))
def test_oracle_algorithmic_bytes_match_instrumented_reference(key):
    if key.startswith("er/"):
        _, n, p, s = key.split("/")
        g = G.er(int(n), float(p), int(s))
    else:
        g = GR.from_edges(G.rmat_edges(10, 16, 1), num_vertices=1 << 10)
    for w, want in BALG[key].items():
        forest, gg = forest_for(w, g)
        _, got = O.run(gg, forest, threads=3)
        assert got == want, (key, w)


def test_survey_balg_numbers():
    # SURVEY.md 8(d) table, produced by the same instrumentation
    assert BALG["er/200/0.1/17"] == {"tc": 227200, "diamond": 409520, "4-cycle": 2354292,
                                     "4-clique": 281764, "5-clique": 283460, "3-motif": 915316}
    assert BALG["rmat/10"]["4-cycle"] == 145863884


@pytest.mark.parametrize("key", sorted(LISTS))
def test_oracle_list_stream_order_matches_reference(key):
    gk, pk, gran = key.split("|")
    _, n, p, s = gk.split("/")
    g = G.er(int(n), float(p), int(s))
    pats = {"triangle": P.generate_clique(3), "4-clique": P.generate_clique(4),
            "diamond": diamond(), "4-cycle": cycle4(),
            "tailed": P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2)], induced="vertex")}
    pat = pats[pk]
    mo, so = analyze(pat, g)
    assert list(mo.order) == LISTS[key]["order"]
    pl = PL.build_plan(pat, mo, so, "list", granularity=gran)
    want = [tuple(m) for m in LISTS[key]["stream"]]
    counts, _, stream = O.run(g, PL.as_forest(pl), threads=1, list_cap=len(want) + 10)
    assert [m for _, m in stream] == want
    assert counts[pat.name] == len(want)
