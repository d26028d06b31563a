"""Binary CSC files straight to HBM (csrc/graph_io.cu).

GGCSR1 files written by the reference's own write_binary load into the same
CSC (and the same run) as an upload of the graph; GGCSR2 round-trips; bad
files fail with the reference read_binary's messages."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle.oracle import Oracle, Reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def need_reference():
    if not Reference.available():
        pytest.skip("oracle/_ref/libggref.so not built")


def _graph(ggb, g):
    return ggb.Graph(g.n, g.off, g.src, g.w, g.outdeg)


def _same_csc(dg, g):
    h = dg.to_host()
    assert h.n == g.n
    assert np.array_equal(h.in_offsets, g.off)
    assert np.array_equal(h.in_sources, g.src)
    assert np.array_equal(h.out_degree, g.outdeg)
    if g.w is not None:
        assert np.array_equal(h.weights, g.w)


def _same_run(ggb, a, b, prog):
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 4, 30, 3)
    ra, rb = ggb.run(a, prog, cfg), ggb.run(b, prog, cfg)
    assert np.array_equal(ra.final_properties, rb.final_properties)
    assert [r.processed_edges for r in ra.per_iteration] == [r.processed_edges for r in rb.per_iteration]


@pytest.mark.parametrize("weighted", [False, True])
def test_reference_ggcsr1_loads(ggb, need_reference, tmp_path, weighted):
    g = Oracle.rmat(14, 16, 5)
    if weighted:
        g.w = Oracle.rmat_weights_u32(g.e, 5).astype(np.float64)
    path = str(tmp_path / "g1.bin")
    Reference.write_binary(g, path)
    dg = ggb.DeviceGraph.load(path)
    _same_csc(dg, g)
    prog = ggb.sssp_spec(0, True) if weighted else ggb.pagerank_spec()
    _same_run(ggb, dg, _graph(ggb, g), prog)
    dg.close()


def test_ggcsr2_round_trip(ggb, tmp_path):
    dg = ggb.DeviceGraph.rmat(15, 16, 7, weights="u32")
    p2 = str(tmp_path / "g2.bin")
    dg.save(p2)
    ref = dg.to_host()
    e = dg.e
    assert os.path.getsize(p2) == 6 + 24 + (dg.n + 1) * 8 + e * 4 + e * 4 + dg.n * 4
    back = ggb.DeviceGraph.load(p2)
    h = back.to_host()
    assert np.array_equal(h.in_offsets, ref.in_offsets)
    assert np.array_equal(h.in_sources, ref.in_sources)
    assert np.array_equal(h.weights, ref.weights)
    assert np.array_equal(h.out_degree, ref.out_degree)
    _same_run(ggb, dg, back, ggb.sssp_spec(3, True))
    dg.close()
    back.close()


def test_bad_files_fail_like_read_binary(ggb, need_reference, tmp_path):
    g = Oracle.rmat(10, 8, 2)
    good = str(tmp_path / "good.bin")
    Reference.write_binary(g, good)
    raw = open(good, "rb").read()
    cases = {
        "magic": b"NOTCSR" + raw[6:],
        "truncated": raw[: len(raw) - 9],
        "source": bytearray(raw),
    }
    n = g.n
    src0 = 30 + (n + 1) * 8  # first source entry of the GGCSR1 layout
    cases["source"][src0:src0 + 8] = int(n + 5).to_bytes(8, "little")
    for name, blob in cases.items():
        p = str(tmp_path / f"{name}.bin")
        open(p, "wb").write(bytes(blob))
        with pytest.raises(RuntimeError) as ref_err:
            Reference.read_binary(p)
        with pytest.raises(RuntimeError) as dev_err:
            ggb.DeviceGraph.load(p)
        assert str(dev_err.value) == str(ref_err.value), name
    with pytest.raises(RuntimeError, match="cannot open binary graph"):
        ggb.DeviceGraph.load(str(tmp_path / "missing.bin"))
