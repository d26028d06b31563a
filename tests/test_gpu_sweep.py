"""Accuracy parity through the reference's sweep protocol, on the device.

The sweep (paper_2104_10039_b200.sweep, bench.cpp:113-227) drives the
device engine; its CSV must equal the reference's golden CSV
(golden_dumbbell4.csv, regenerated from the reference as
tests/golden/dumbbell4_sweep.csv), and on the acceptance suite's PR
workload (power-law 10k, acceptance_main.cpp:64-77) every cell's accuracy
and edge ratio must equal the oracle-driven sweep's (and the recorded
reference numbers, test_output.txt:10-15)."""
import os

import numpy as np

import pytest

from oracle.oracle import Oracle
from tests.parity import oracle_runner

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_device_sweep_reproduces_golden_csv(ggb):
    from paper_2104_10039_b200 import sweep
    d = Oracle.dumbbell(4)
    plan = sweep.SweepPlan(algo="wcc", graph=ggb.Graph(d.n, d.off, d.src),
                           graph_label="gen:dumbbell:4", schemes=["sp", "gg"],
                           sigma_grid=[0.4, 0.8], theta_grid=[0.5], alpha_grid=[2], iterations=16,
                           repeats=1, seeds=[1, 2])
    ours = sweep.mask_time_columns(sweep.emit_csv(sweep.run_sweep(plan), plan))
    with open(os.path.join(GOLDEN, "dumbbell4_sweep.csv")) as f:
        assert ours == sweep.mask_time_columns(f.read())


def _pr10k_plan(ggb, **kw):  # acceptance_main.cpp:64-77
    from paper_2104_10039_b200 import sweep
    g = Oracle.power_law(10000, 16.0, 2.1, 7)
    plan = sweep.SweepPlan(algo="pr", graph=ggb.Graph(g.n, g.off, g.src),
                           graph_label="gen:powerlaw:10000,16,2.1", iterations=50, epsilon=1e-9,
                           repeats=1, seeds=[1, 2, 3, 4, 5], threads=2, schemes=["gg"])
    for k, v in kw.items():
        setattr(plan, k, v)
    return plan


def _rows_equal(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert (x.scheme, x.sigma, x.theta, x.alpha, x.iters) == (y.scheme, y.sigma, y.theta, y.alpha, y.iters)
        # top-k errors are exact integer counts; relative / stretch errors are
        # sums the device reduces in a fixed tree order (metrics.cu), equal to
        # the reference's left-to-right sum up to rounding
        assert x.accuracy == pytest.approx(y.accuracy, rel=1e-12, abs=1e-12), (x, y)
        assert x.edge_ratio == y.edge_ratio, (x, y)


def test_sigma_monotonicity_cells_equal_oracle(ggb):  # acceptance criterion 4
    from paper_2104_10039_b200 import sweep
    plan = _pr10k_plan(ggb, sigma_grid=[0.1, 0.3, 0.5, 0.7, 0.9], theta_grid=[0.1], alpha_grid=[5])
    dev = sweep.run_sweep(plan)
    _rows_equal(dev, sweep.run_sweep(plan, runner=oracle_runner))
    gg = [r for r in dev if r.scheme == "gg"]
    assert gg[0].accuracy == pytest.approx(13.8) and gg[-1].accuracy == pytest.approx(25.6)


def test_work_reduction_band_equal_oracle(ggb):  # acceptance criterion 9
    from paper_2104_10039_b200 import sweep
    plan = _pr10k_plan(ggb, sigma_grid=[0.2, 0.3, 0.5], theta_grid=[0.005, 0.01, 0.02], alpha_grid=[5])
    dev = sweep.run_sweep(plan)
    _rows_equal(dev, sweep.run_sweep(plan, runner=oracle_runner))
    hit = [r for r in dev if r.scheme == "gg" and 90.0 <= r.accuracy <= 95.0 and r.edge_ratio < 0.75]
    best = min(hit, key=lambda r: r.edge_ratio)
    assert (best.sigma, best.theta, best.alpha) == (0.2, 0.01, 5)
    assert best.accuracy == pytest.approx(90.8) and best.edge_ratio == pytest.approx(0.469386, abs=1e-6)


def _find(rows, scheme, sigma, theta, alpha):  # acceptance_main.cpp:54-63
    hit = [r for r in rows if (r.scheme, r.sigma, r.theta, r.alpha) == (scheme, sigma, theta, alpha)]
    assert len(hit) == 1
    return hit[0]


def test_theta_tradeoff_equal_oracle(ggb):  # acceptance criterion 5
    from paper_2104_10039_b200 import sweep
    plan = _pr10k_plan(ggb, sigma_grid=[0.5], theta_grid=[0.05, 0.5, 0.8], alpha_grid=[5])
    dev = sweep.run_sweep(plan)
    _rows_equal(dev, sweep.run_sweep(plan, runner=oracle_runner))
    lo, mid, hi = (_find(dev, "gg", 0.5, t, 5) for t in (0.05, 0.5, 0.8))
    # test_output.txt:11: accuracy 37.2 / 6.8 / 4, ratio 0.529138 / 0.38515 / 0.370695
    assert (lo.accuracy, mid.accuracy, hi.accuracy) == pytest.approx((37.2, 6.8, 4.0))
    assert (lo.edge_ratio, mid.edge_ratio, hi.edge_ratio) == \
        pytest.approx((0.529138, 0.38515, 0.370695), abs=1e-6)
    assert lo.accuracy >= mid.accuracy >= hi.accuracy
    assert lo.edge_ratio > mid.edge_ratio >= hi.edge_ratio


@pytest.mark.parametrize("algo", ["pr", "sssp"])
def test_between_sp_and_sms_reproduces_reference(ggb, algo):  # acceptance criterion 6
    """The reference's own known-red criterion (acceptance_main.cpp:262-300):
    the device sweep reproduces the reference's numbers, including the
    violation the reference documents."""
    from paper_2104_10039_b200 import sweep
    plan = _pr10k_plan(ggb, algo=algo, epsilon=-1.0, schemes=["sp", "sms", "gg"], sigma_grid=[0.5],
                       theta_grid=[0.5], alpha_grid=[5])
    if algo == "sssp":
        plan.iterations = 0  # the accurate reference runs to convergence
    dev = sweep.run_sweep(plan)
    _rows_equal(dev, sweep.run_sweep(plan, runner=oracle_runner))
    sp, sms, gg = _find(dev, "sp", 0.5, 0.0, 0), _find(dev, "sms", 0.5, 0.5, 5), _find(dev, "gg", 0.5, 0.5, 5)
    ref = {"pr": ((80.8, 6.8, 97.0), (0.499263, 0.384592, 0.743478)),  # test_output.txt:12
           "sssp": ((65.675, 66.5343, 74.6464), (0.499263, 0.408551, 0.706209))}[algo]
    assert (sp.accuracy, gg.accuracy, sms.accuracy) == pytest.approx(ref[0], abs=5e-5 * 100)
    assert (sp.edge_ratio, gg.edge_ratio, sms.edge_ratio) == pytest.approx(ref[1], abs=1e-6)


def test_wcc_gg_equals_sms(ggb):  # acceptance criterion 7 (acceptance_main.cpp:304-326)
    for seed in range(1, 11):
        g = Oracle.symmetrized(Oracle.power_law(400, 5.0, 2.2, seed))
        graph = ggb.Graph(g.n, g.off, g.src)
        a = ggb.run(graph, ggb.wcc_spec(), ggb.EngineConfig("gg", 0.5, 0.5, 2, 64, seed))
        b = ggb.run(graph, ggb.wcc_spec(), ggb.EngineConfig("sms", 0.5, 0.5, 2, 64, seed))
        assert (a.final_properties == b.final_properties).all(), seed


@pytest.mark.parametrize("kind", ["rmat", "random_weighted"])
def test_device_symmetrized_equals_reference_order(ggb, kind):
    """gg_dev_graph_symmetrized reproduces graph.cpp:249-257 exactly: per
    destination its in-edges in CSC order, then its out-edges' reversals in
    ascending edge id (the order decides WCC influences and masks)."""
    if kind == "rmat":
        dg = ggb.DeviceGraph.rmat(12, 16, 3)
        g = Oracle.rmat(12, 16, 3)
    else:
        g = Oracle.random_graph(3000, 40000, 4, True)  # in-lists in edge order, not sorted
        dg = ggb.DeviceGraph.upload(ggb.Graph(g.n, g.off, g.src, g.w))
        dg.weight_dtype = np.float64
    sym = dg.symmetrized()
    h = sym.to_host()
    ref = Oracle.symmetrized(g)
    assert np.array_equal(h.in_offsets, ref.off)
    assert np.array_equal(h.in_sources, ref.src)
    assert np.array_equal(h.out_degree, ref.outdeg)
    if kind != "rmat":
        assert np.array_equal(h.weights, ref.w)
    sym.close()
    dg.close()


def test_c1_sweep_on_resident_graph_equals_oracle(ggb):
    """The sweep protocol on a resident device graph (BASELINE c1: PR on
    R-MAT s16), cells equal to the oracle-driven sweep on its host copy."""
    from paper_2104_10039_b200 import sweep
    dg = ggb.DeviceGraph.rmat(16, 16, 1)
    host = dg.to_host()
    kw = dict(algo="pr", graph_label="rmat:16,16,1", schemes=["sp", "gg"], sigma_grid=[0.3, 0.5],
              theta_grid=[0.01, 0.1], alpha_grid=[4], repeats=1, seeds=[1, 2], threads=4)
    dev = sweep.run_sweep(sweep.SweepPlan(graph=dg, **kw))
    orc = sweep.run_sweep(sweep.SweepPlan(graph=host, **kw), runner=oracle_runner)
    _rows_equal(dev, orc)
    dg.close()
