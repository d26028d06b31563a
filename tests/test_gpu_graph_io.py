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


def _ranks(ggb, fn, nranks):
    """fn(rank, exchange handle) on nranks host threads (in-process transport)."""
    import threading
    xs = ggb.Exchange.local_group(nranks)
    out, errs = [None] * nranks, [None] * nranks

    def work(r):
        try:
            out[r] = fn(r, xs[r].handle)
        except BaseException as e:  # noqa: BLE001 - returned to the caller
            errs[r] = e
    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for x in xs:
        x.close()
    return out, errs


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_ggcsr2_stored_out_degrees_are_validated(ggb, tmp_path, nranks):
    """GGCSR2 carries the out-degrees; a file whose stored degrees are not
    the sources' counts is rejected with Graph::validate's message
    (graph.cpp:88-93), also when each rank holds only a slice of the
    sources (the counts are summed over ranks)."""
    dg = ggb.DeviceGraph.rmat(12, 8, 9)
    good = str(tmp_path / "good2.bin")
    dg.save(good)
    n, e = dg.n, dg.e
    dg.close()
    raw = bytearray(open(good, "rb").read())
    deg0 = 6 + 24 + (n + 1) * 8 + e * 4  # first stored out-degree (unweighted GGCSR2)
    v = 5
    d = int.from_bytes(raw[deg0 + 4 * v: deg0 + 4 * v + 4], "little")
    raw[deg0 + 4 * v: deg0 + 4 * v + 4] = (d + 1).to_bytes(4, "little")
    bad = str(tmp_path / "bad2.bin")
    open(bad, "wb").write(bytes(raw))

    def load(path):
        def fn(r, x):
            g = ggb.DeviceGraph.load(path, device=0, rank=r, nranks=nranks, exchange=x) \
                if nranks > 1 else ggb.DeviceGraph.load(path)
            g.close()
            return True
        return _ranks(ggb, fn, nranks)
    ok, errs = load(good)
    assert all(ok) and not any(errs)
    _, errs = load(bad)
    assert all(errs)
    for err in errs:
        assert str(err) == "graph: out_degree inconsistent with edges"


def test_create_validates_sources_and_offsets(ggb):
    """gg_dev_graph_create on a host CSC view: a source >= n (also when the
    caller supplies out-degrees) and decreasing offsets fail creation with
    Graph::validate's conditions (graph.cpp:83-92) instead of reading out of
    bounds on the device."""
    n = 6
    off = np.array([0, 2, 3, 3, 5, 6, 7], np.uint64)
    src = np.array([1, 2, 0, 5, 1, 3, 4], np.uint32)
    deg = np.bincount(src, minlength=n).astype(np.uint32)
    ggb.DeviceGraph.upload(ggb.Graph(n, off, src, None, deg)).close()  # valid
    bad_src = src.copy()
    bad_src[4] = n + 3
    with pytest.raises(ValueError, match="edge source out of range"):
        ggb.DeviceGraph.upload(ggb.Graph(n, off, bad_src, None, deg))
    bad_off = off.copy()
    bad_off[2], bad_off[3] = 4, 3  # 2, 4, 3: decreases (offsets[n] still == e)
    with pytest.raises(ValueError, match="offsets decrease"):
        ggb.DeviceGraph.upload(ggb.Graph(n, bad_off, src, None, deg))
