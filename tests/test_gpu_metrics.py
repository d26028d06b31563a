"""Device error metrics (csrc/metrics.cu) against the reference's own
metrics.cpp (oracle/_ref) and the host implementations: top-k exact (ties
broken by ascending vertex, -0.0 == +0.0), relative / stretch within 1e-12
(fixed-order device reduction vs the reference's left-to-right sum), the
stretch abort naming the same vertex; and the sweep pattern: metrics of two
runs' device projections equal the metrics of their host exports."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import Reference

pytestmark = pytest.mark.gpu


def _dev(ggb, x):
    return ggb.DeviceBuffer.upload(np.ascontiguousarray(x, np.float64))


@pytest.fixture(scope="module")
def need_reference():
    if not Reference.available():
        pytest.skip("oracle/_ref/libggref.so not built")


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_topk_matches_reference_with_ties(ggb, need_reference, seed):
    rng = np.random.default_rng(seed)
    n = 50_000
    exact = rng.integers(0, 40, n).astype(np.float64) / 7.0  # heavy ties
    approx = exact + rng.normal(0, 0.05, n) * (rng.random(n) < 0.3)
    exact[rng.integers(0, n, 50)] = -0.0
    approx[rng.integers(0, n, 50)] = 0.0
    for k in (1, 17, 500, 4999, n):
        ref = Reference.metric(0, approx, exact, k)
        dev = ggb.topk_error(_dev(ggb, approx), _dev(ggb, exact), k)
        host = ggb.topk_error(approx, exact, k)
        assert dev.error == ref == host.error, (k, dev.error, ref, host.error)


@pytest.mark.parametrize("seed", [4, 5])
def test_relative_and_stretch_match_reference(ggb, need_reference, seed):
    rng = np.random.default_rng(seed)
    n = 200_003
    exact = rng.integers(0, 1000, n).astype(np.float64)
    exact[rng.integers(0, n, 1000)] = np.inf  # unreachable
    exact[7] = 0.0                             # the source
    approx = exact.copy()
    bump = rng.random(n) < 0.2
    approx[bump] += rng.integers(1, 50, int(bump.sum()))
    approx[rng.integers(0, n, 500)] = np.inf   # reachable exactly, lost approximately
    approx[7] = 0.0
    a, x = _dev(ggb, approx), _dev(ggb, exact)
    for which, fn in ((1, ggb.relative_error), (2, ggb.stretch_error)):
        ref = Reference.metric(which, approx, exact)
        dev = fn(a, x).error
        assert dev == pytest.approx(ref, rel=1e-12, abs=1e-15), (which, dev, ref)


def test_stretch_abort_names_the_vertex(ggb):
    exact = np.array([0.0, 3.0, 5.0, 2.0, 9.0])
    approx = np.array([0.0, 3.0, 4.0, 1.0, 9.0])  # vertices 2 and 3 below exact
    with pytest.raises(RuntimeError, match="at vertex 2 "):
        ggb.stretch_error(_dev(ggb, approx), _dev(ggb, exact))


def test_sweep_projection_metrics(ggb):
    dg = ggb.DeviceGraph.rmat(15, 16, 9)
    pr = ggb.pagerank_spec(0.85, 1e-7)
    exact_rep = ggb.run(dg, pr, ggb.EngineConfig("accurate", max_iterations=40))
    exact_dev = ggb.DeviceBuffer.copy(dg.last_projection())
    approx_rep = ggb.run(dg, pr, ggb.EngineConfig("gg", 0.5, 0.01, 4, exact_rep.iterations_run, 9))
    approx_dev = dg.last_projection()
    k = max(1, dg.n // 100)
    assert ggb.topk_error(approx_dev, exact_dev, k).error == \
        ggb.topk_error(approx_rep.final_properties, exact_rep.final_properties, k).error
    assert ggb.relative_error(approx_dev, exact_dev).error == pytest.approx(
        ggb.relative_error(approx_rep.final_properties, exact_rep.final_properties).error,
        rel=1e-12)
    exact_dev.close()
    dg.close()
