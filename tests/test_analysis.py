"""Analyzer + plan IR equal the reference's, pinned by tests/golden/analysis.json
(reference pattern.py / plan.py outputs for 70+ patterns and 4 graph stats)."""
import json
from pathlib import Path

import pytest

from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import plan as PL

GOLD = json.loads((Path(__file__).parent / "golden" / "analysis.json").read_text())


def _pattern(rec):
    return P.Pattern(rec["size"], [tuple(e) for e in rec["edges"]], labels=rec["labels"],
                     induced=rec["induced"], name=rec["name"])


def _stats(s):
    return None if s is None else P.GraphStats(avg_degree=s[0], num_vertices=s[1])


@pytest.mark.parametrize("key", sorted(GOLD["patterns"]))
def test_pattern_analysis_matches_reference(key):
    rec = GOLD["patterns"][key]
    p = _pattern(rec)
    unnamed = P.Pattern(rec["size"], [tuple(e) for e in rec["edges"]], labels=rec["labels"],
                        induced=rec["induced"])
    if not key.startswith("motif"):   # motifs are renamed by generate_all_motifs
        assert unnamed.name == rec["name"]
    assert repr(p.canonical_form()) == rec["canonical"]
    assert sorted(list(a) for a in P.automorphisms(p)) == rec["auts"]
    orders = [[list(mo.order), [sorted(c) for c in mo.conn], [sorted(a) for a in mo.anti]]
              for mo in P.enumerate_matching_orders(p)]
    assert orders == rec["orders"]
    for r in rec["per_stats"]:
        st = _stats(r["stats"])
        mo = P.select_matching_order(P.enumerate_matching_orders(p), st)
        so = P.generate_symmetry_order(p, mo)
        props = P.detect_properties(p, mo, so)
        assert list(mo.order) == r["order"]
        assert sorted(list(c) for c in so.constraints) == r["symmetry"]
        assert [props.is_clique, sorted(props.hub_vertices),
                None if props.decomposition is None else list(props.decomposition),
                props.automorphism_count] == r["props"]
        assert P.describe_analysis(p, mo, so) == r["describe"]
        for pk, text in r["plans"].items():
            parts = pk.split("/")
            mode, gran, oriented = parts[0], parts[1], bool(int(parts[2]))
            pl = PL.build_plan(p, mo, so, mode, granularity=gran, oriented=oriented)
            if len(parts) == 4:
                pl = PL.apply_counting_rewrite(pl, props)
            assert PL.emit_source(PL.as_forest(pl)) == text, (key, pk)


def test_motif_names_match_reference():
    for k, names in GOLD["motif_names"].items():
        assert [p.name for p in P.generate_all_motifs(int(k))] == names


@pytest.mark.parametrize("key", sorted(GOLD["fused"]))
def test_fused_forests_match_reference(key):
    k, gran, mode = key.split("/")
    plans = []
    for p in P.generate_all_motifs(int(k)):
        mo = P.select_matching_order(P.enumerate_matching_orders(p))
        so = P.generate_symmetry_order(p, mo)
        pl = PL.build_plan(p, mo, so, mode, granularity=gran)
        if mode == "count":
            pl = PL.apply_counting_rewrite(pl, P.detect_properties(p, mo, so))
        plans.append(pl)
    assert PL.emit_source(PL.fuse_multi_pattern(plans)) == GOLD["fused"][key]


def test_validation_errors():
    with pytest.raises(ValueError, match="maximum"):
        P.Pattern(9, [(i, i + 1) for i in range(8)])
    with pytest.raises(ValueError, match="connected"):
        P.Pattern(4, [(0, 1), (2, 3)])
    with pytest.raises(ValueError):
        P.generate_clique(9)
    with pytest.raises(ValueError):
        P.generate_all_motifs(6)
    d = P.Pattern(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3)])
    mo = P.select_matching_order(P.enumerate_matching_orders(d))
    so = P.generate_symmetry_order(d, mo)
    with pytest.raises(ValueError):
        PL.build_plan(d, mo, so, "stream")
    with pytest.raises(ValueError):
        PL.build_plan(d, mo, so, "count", oriented=True)
    with pytest.raises(ValueError):
        PL.apply_counting_rewrite(PL.build_plan(d, mo, so, "list"), P.detect_properties(d, mo, so))


def test_parse_pattern(tmp_path):
    f = tmp_path / "c4.el"
    f.write_text("0 1\n1 2\n2 3\n3 0\n")
    p = P.parse_pattern(str(f))
    assert p.size == 4 and p.num_edges == 4 and p.name == "4-cycle"
