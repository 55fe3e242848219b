"""GCSR v1 binary IO against files written by the reference's own
``save_csr`` (graph.py:293-323; fixtures from tests/golden/make_gcsr.py):
the CPU reference and this package load the identical graph file."""
from pathlib import Path

import numpy as np
import pytest

import graphs as G
import paper_2112_09761_b200 as pm
from paper_2112_09761_b200 import graph as GR

GOLD = Path(__file__).resolve().parent / "golden"
DATA = Path(__file__).resolve().parent / "data"


def _ours(name):
    if name == "k4_labeled":
        return pm.load_edgelist(str(DATA / "k4.el"), labeled=True, label_path=str(DATA / "k4.el.labels"))
    if name == "er60_oriented":
        e, _ = G.er_edges(60, 0.2, 3)
        return _orient_host(GR.from_edges(e, num_vertices=60))
    return GR.from_edges(G.rmat_edges(8, 16, 1), num_vertices=256)


def _orient_host(g):
    from util import orient_host
    return orient_host(g)


@pytest.mark.parametrize("name", ["k4_labeled", "er60_oriented", "rmat8"])
def test_load_reference_file_and_rewrite_identical(name, tmp_path):
    ref = (GOLD / f"{name}.gcsr").read_bytes()
    g = pm.load_csr(str(GOLD / f"{name}.gcsr"))
    g.validate()
    out = tmp_path / "x.gcsr"
    pm.save_csr(g, str(out))
    assert out.read_bytes() == ref


@pytest.mark.parametrize("name", ["k4_labeled", "er60_oriented", "rmat8"])
def test_host_builders_write_the_reference_bytes(name, tmp_path):
    g = _ours(name)
    out = tmp_path / "x.gcsr"
    pm.save_csr(g, str(out))
    assert out.read_bytes() == (GOLD / f"{name}.gcsr").read_bytes()


def test_header_layout():
    b = (GOLD / "k4_labeled.gcsr").read_bytes()
    assert b[:4] == b"GCSR"
    ver, nv, ne, flags = np.frombuffer(b[4:8], "<u4")[0], *np.frombuffer(b[8:24], "<u8"), \
        np.frombuffer(b[24:28], "<u4")[0]
    assert (ver, nv, ne, flags) == (1, 4, 12, 1)
    assert len(b) == 28 + 8 * (nv + 1) + 4 * ne + 4 * nv


def test_bad_magic_and_version(tmp_path):
    p = tmp_path / "bad.gcsr"
    p.write_bytes(b"XXXX" + bytes(24))
    with pytest.raises(ValueError, match="magic"):
        pm.load_csr(str(p))
    b = bytearray((GOLD / "rmat8.gcsr").read_bytes())
    b[4] = 2
    p.write_bytes(bytes(b))
    with pytest.raises(ValueError, match="version"):
        pm.load_csr(str(p))


@pytest.mark.gpu
def test_device_built_graph_exports_reference_bytes(tmp_path):
    # device CSR builder (and device orientation) -> GCSR: byte-identical to
    # the reference's file of the same input
    g = GR.from_edges_device(G.rmat_edges(8, 16, 1), num_vertices=256)
    out = tmp_path / "d.gcsr"
    pm.save_csr(g, str(out))
    assert out.read_bytes() == (GOLD / "rmat8.gcsr").read_bytes()
    e, _ = G.er_edges(60, 0.2, 3)
    og = pm.orient(GR.from_edges_device(e, num_vertices=60))
    pm.save_csr(og, str(out))
    assert out.read_bytes() == (GOLD / "er60_oriented.gcsr").read_bytes()
