"""Generated bitmap local-graph-search kernels for hub-rooted plans
(codegen_lgs; reference _LocalRunner / run_dfs_lgs, executor.py:415-599):
which plans qualify, and that every kernel compiles for sm_100a (NVRTC, no
GPU needed). GPU parity is in test_gpu_lgs.py."""
import pytest

from paper_2112_09761_b200 import codegen_lgs as CL
from paper_2112_09761_b200 import executor as EX
from paper_2112_09761_b200 import pattern as P
from util import TAILED_EDGES, diamond, make_plan

BOOK = P.Pattern(5, [(0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (0, 4), (1, 4)])
STAR3 = P.Pattern(4, [(0, 1), (0, 2), (0, 3)])
WEDGE = P.Pattern(3, [(0, 1), (0, 2)])


def hub_plans():
    out = {}
    for gran in ("edge", "vertex"):
        for mode in ("count", "list"):
            out[f"diamond-{mode}-{gran}"] = make_plan(diamond(), mode=mode, granularity=gran)
    out["book-list-edge"] = make_plan(BOOK, mode="list")
    out["tailed-list-vertex"] = make_plan(P.Pattern(4, TAILED_EDGES), mode="list", granularity="vertex")
    out["3-star-list"] = make_plan(STAR3, mode="list", granularity="vertex")
    out["wedge-count"] = make_plan(WEDGE, granularity="vertex")
    out["6-clique-count"] = make_plan(P.generate_clique(6), oriented=True)
    out["8-clique-list-vertex"] = make_plan(P.generate_clique(8), mode="list", granularity="vertex", oriented=True)
    out["diamond-rewrite"] = make_plan(diamond(), rewrite=True)
    return out


def test_hub_rootedness_of_the_fixtures():
    for name, pl in hub_plans().items():
        p = pl.pattern
        assert p.degree(pl.matching_order.order[0]) == p.size - 1, name


@pytest.mark.parametrize("name", sorted(hub_plans()))
def test_lgs_kernel_compiles(name):
    pl = hub_plans()[name]
    if pl.parallel_granularity == "edge" and pl.pattern.degree(pl.matching_order.order[1]) != pl.pattern.size - 1:
        pytest.skip("edge LGS needs hubs at levels 1 and 2")
    for maxdeg in ((40, 3000) if name.startswith("diamond-list") else (200,)):
        cp = EX.compile_lgs(pl, list_mode=pl.mode == "list", max_degree=maxdeg)
        assert cp.handle
        assert cp.gen.max_level == pl.depth
        assert (cp.gen.num_slots == 0) == (CL.lgs_ncap(maxdeg) <= CL.SMEM_NCAP)


def test_needs_rows():
    assert not CL.needs_rows(make_plan(WEDGE, granularity="vertex"))
    assert CL.needs_rows(make_plan(STAR3, granularity="vertex"))   # a buffered non-anchored level
    assert CL.needs_rows(make_plan(diamond()))
    assert not CL.needs_rows(make_plan(P.generate_clique(3), oriented=True))
    assert CL.needs_rows(make_plan(P.generate_clique(4), oriented=True))
