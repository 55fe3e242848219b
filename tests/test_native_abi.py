"""libg2m.so loads without a GPU, exports every symbol include/g2m.h declares,
and NVRTC compiles the generated sm_100a kernels (no device needed)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2112_09761_b200 import _native as N
from paper_2112_09761_b200 import executor as EX
from paper_2112_09761_b200 import pattern as P
from paper_2112_09761_b200 import plan as PL
from util import cycle4, diamond, make_plan

HEADER = Path(__file__).resolve().parent.parent / "include" / "g2m.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:const char\*|int32_t|int)\s+(g2m_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.SIGNATURES)
    assert lib.g2m_abi_version() == N.ABI_VERSION == 7


def test_struct_layouts():
    assert C.sizeof(N.TaskSpec) == 48
    assert C.sizeof(N.KernelMeta) == 64
    assert C.sizeof(N.RunStats) == 8 * 16 + 24


def _forests():
    out = {
        "tc": PL.as_forest(make_plan(P.generate_clique(3), oriented=True)),
        "4-clique": PL.as_forest(make_plan(P.generate_clique(4), oriented=True)),
        "5-clique": PL.as_forest(make_plan(P.generate_clique(5), oriented=True)),
        "4-cycle": PL.as_forest(make_plan(cycle4())),
        "diamond": PL.as_forest(make_plan(diamond(), rewrite=True)),
        "diamond-list": PL.as_forest(make_plan(diamond(), mode="list")),
    }
    plans = [make_plan(p, granularity="vertex", rewrite=True) for p in P.generate_all_motifs(3)]
    out["3-motif"] = PL.fuse_multi_pattern(plans)
    plans = [make_plan(p, rewrite=True) for p in P.generate_all_motifs(4)]
    out["4-motif"] = PL.fuse_multi_pattern(plans)
    return out


@pytest.mark.parametrize("name", sorted(_forests()))
def test_nvrtc_compiles_generated_kernel(name):
    forest = _forests()[name]
    for list_mode in (False, True):
        for maxdeg in (100, 10 ** 6):
            cp = EX.compile_forest(forest, labeled=False, list_mode=list_mode, max_degree=maxdeg)
            assert cp.handle
            assert EX.codegen.KERNEL_NAME in cp.gen.source


def test_no_gpu_path_raises():
    if N.device_count() > 0:
        pytest.skip("GPU present")
    import graphs as G
    import paper_2112_09761_b200 as pm
    with pytest.raises(N.NativeUnavailable):
        pm.triangle_count(G.complete(4))


@pytest.mark.parametrize("name", ["4-motif", "4-cycle", "diamond-list", "5-clique"])
def test_nvrtc_compiles_frontier_kernels(name):
    """The bounded-frontier BFS expand/consume pair compiles for every forest
    with a level-3 subtree (and is refused for the others)."""
    forest = _forests()[name]
    if EX.codegen.frontier_nodes(forest) == 0 or forest.uses_orientation:
        pytest.skip("no level-3 subtree on an edge-parallel forest")
    for fr in ("expand", "consume"):
        cp = EX.compile_forest(forest, labeled=False, list_mode=False, max_degree=1000, frontier=fr)
        assert cp.handle
    with pytest.raises(ValueError):
        EX.codegen.generate(forest, labeled=True, frontier="expand")


def test_search_chooser():
    import graphs as G
    g = G.er(60, 0.2, 3)
    plans = [make_plan(p, rewrite=True) for p in P.generate_all_motifs(4)]
    f = PL.fuse_multi_pattern(plans)
    tasks = EX._default_tasks(g, f)
    assert EX.choose_search(g, f, tasks, EX.ExecutionConfig(search="dfs"))[0] == "dfs"
    assert EX.choose_search(g, f, tasks, EX.ExecutionConfig(search="bfs"))[0] == "bfs"
    # ER is not skewed: auto keeps DFS
    assert EX.choose_search(g, f, tasks)[0] == "dfs"
    from paper_2112_09761_b200 import graph as GRM
    hub = GRM.from_edges([(0, i) for i in range(1, 400)] + [(i, i + 1) for i in range(1, 399)],
                         num_vertices=400)          # max degree 399 >> average 4
    assert EX.choose_search(hub, f, EX._default_tasks(hub, f))[0] == "bfs"
    assert EX.choose_search(hub, f, EX._default_tasks(hub, f),
                            EX.ExecutionConfig(frontier_bytes=64))[0] == "dfs"
    tc = PL.as_forest(make_plan(P.generate_clique(3), oriented=True))
    assert EX.choose_search(g, tc, EX._default_tasks(g, tc))[0] == "dfs"
    with pytest.raises(ValueError):
        EX.choose_search(g, f, tasks, EX.ExecutionConfig(search="nope"))
