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
    assert lib.g2m_abi_version() == 2


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
