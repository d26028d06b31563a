"""Pins the CPU oracle (oracle/gg_oracle.c) to the reference (CPU tests).

1. every golden run in tests/golden/reference_runs.json (generated from the
   reference itself by tests/golden/make_golden.py) is reproduced bit for bit;
2. the reference's known-answer tests (test_engine.cpp, test_algorithms.cpp,
   acceptance_main.cpp) hold on the oracle;
3. when oracle/_ref/libggref.so is present, the oracle equals the live
   reference on further seeded inputs;
4. the sweep protocol driven by the oracle reproduces the reference's
   golden CSV (golden_dumbbell4.csv, regenerated from the reference as
   tests/golden/dumbbell4_sweep.csv).
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import (ACCURATE, BP, BP_EDGE, GG, PR, SMS, SP, SSSP, WCC, Oracle,
                           Reference)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "reference_runs.json")) as f:
        return json.load(f)


def _graph(kind, p):
    if kind == "dumbbell":
        return Oracle.dumbbell(p["k"])
    if kind == "power_law":
        return Oracle.power_law(p["n"], p["avg"], p["ex"], p["seed"])
    if kind == "random":
        return Oracle.random_graph(p["n"], p["m"], p["seed"], p["weighted"])
    raise ValueError(kind)


def test_oracle_generators_match_golden(golden):
    for name, meta in golden["graphs"].items():
        if meta["kind"] == "rmat_bpedge":
            continue
        g = _graph(meta["kind"], meta["params"])
        assert (g.n, g.e) == (meta["n"], meta["e"]), name
        assert int(g.src.astype(np.int64).sum()) == meta["src_sum"], name
        assert int(g.off.astype(np.int64).sum()) == meta["off_sum"], name


def test_oracle_reproduces_reference_runs(golden):
    cache = {}
    for run in golden["runs"]:
        name = run["graph"]
        if name == "rmat9_s4_bpedge":
            g = Oracle.rmat(9, 16, 4)
            c = Oracle.bp_couplings(g.e, 4)
            dst = np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64)))
            graph = Oracle.build_graph(g.n, g.src, dst, c.astype(np.float64))
            pp = dict(prior_table=Oracle.bp_priors(g.n, 4))
        else:
            meta = golden["graphs"][name]
            if name not in cache:
                g = _graph(meta["kind"], meta["params"])
                cache[name] = (g, Oracle.symmetrized(g))
            graph = cache[name][1] if run["prog"] == WCC else cache[name][0]
            pp = dict(run["params"])
        r = Oracle.run(graph, run["prog"], **run["config"], **pp)
        ctx = (name, run["prog"], run["params"], run["config"])
        assert r.status == run["status"], ctx
        assert r.iterations_run == run["iterations_run"], ctx
        assert r.modes == run["modes"], ctx
        assert r.processed_edges == run["processed_edges"], ctx
        assert r.active_vertices == run["active_vertices"], ctx
        if run["prog"] == WCC:
            assert [int(x) for x in r.props] == run["props"], ctx
        else:
            assert [float(x).hex() for x in r.props.reshape(-1)] == run["props"], ctx


def test_sparsify_known_answers(golden):  # test_engine.cpp:54-80
    g = Oracle.random_graph(40, 500, 1)
    assert int(Oracle.sparsify(g.e, 1.0, 9).sum()) == g.e
    assert int(Oracle.sparsify(g.e, 0.0, 9).sum()) == 0
    with pytest.raises(ValueError):
        Oracle.sparsify(g.e, 1.2, 9)
    cnt = int(Oracle.sparsify(100000, 0.5, 3).sum())
    assert 49000 <= cnt <= 51000 and cnt == golden["sparsify_e100000_s3_popcount"]
    a, b = Oracle.sparsify(2000, 0.3, 5), Oracle.sparsify(2000, 0.7, 5)
    assert np.all(b[a == 1] == 1)
    assert "".join(str(int(x)) for x in a) == golden["sparsify_e2000_prefix"]["bits"]


def test_schedule_known_answers():  # test_engine.cpp:82-103
    assert Oracle.supersteps(2, 10, GG) == [3, 6, 9]
    assert Oracle.supersteps(4, 3, SMS) == []
    assert Oracle.supersteps(1, 4, GG) == [2, 4]
    assert Oracle.supersteps(4, 10, SMS) == [5]
    assert Oracle.supersteps(2, 10, ACCURATE) == [] and Oracle.supersteps(2, 10, SP) == []
    for s in (SMS, GG):
        sup = Oracle.supersteps(3, 20, s)
        for t in range(1, 21):
            assert (Oracle.mode_for(s, t, 3) == 2) == (t in sup)
    assert Oracle.mode_for(SMS, 10, 3) == 1 and Oracle.mode_for(SP, 10, 3) == 0


def test_engine_known_answers():
    # test_engine.cpp:122-131 sp sigma 0 leak
    r = Oracle.run(Oracle.dumbbell(2), PR, scheme=SP, sigma=0.0, max_iterations=50)
    np.testing.assert_allclose(r.props, 0.15 / 4, rtol=1e-12)
    assert r.iterations_run == 2
    # :184-194 early exit
    c4 = Oracle.build_graph(4, [0, 1, 2, 3], [1, 2, 3, 0])
    r = Oracle.run(c4, PR, max_iterations=100)
    assert r.iterations_run == 1
    # :226-237 3-cycle gathers every edge
    r = Oracle.run(Oracle.build_graph(3, [0, 1, 2], [1, 2, 0]), PR, max_iterations=5, epsilon=1e-15)
    assert all(x == 3 for x in r.processed_edges) and all(x == 3 for x in r.active_vertices)
    # :239-256 unreachable theta
    r = Oracle.run(Oracle.dumbbell(3), PR, scheme=GG, sigma=1.0, theta=2.0, alpha=5, max_iterations=10)
    assert r.modes[5] == 2 and all(m == 0 for m in r.modes[6:]) and all(e == 0 for e in r.processed_edges[6:])
    np.testing.assert_allclose(r.props, 0.15 / 6, rtol=1e-12)
    # :288-302 NaN abort
    r = Oracle.run(c4, 5, max_iterations=50)
    assert r.status == 2 and (r.err_iteration, r.err_vertex) == (3, 2)
    assert "iteration 3" in r.msg and "vertex 2" in r.msg
    # :304-309 empty graph
    r = Oracle.run(Oracle.build_graph(0, [], []), PR)
    assert r.iterations_run == 0
    # :105-120 config validation
    assert Oracle.run(c4, PR, sigma=1.5).msg == "sigma must be in [0,1]"
    assert Oracle.run(c4, PR, sigma=0.5, alpha=0).msg == "alpha must be >= 1"
    assert Oracle.run(c4, PR, threads=0).status == 1
    assert Oracle.run(c4, PR, max_iterations=0).status == 1


def test_algorithm_known_answers():  # test_algorithms.cpp
    star = Oracle.build_graph(4, [0, 1, 2], [3, 3, 3])
    r = Oracle.run(star, PR, max_iterations=300, epsilon=1e-16)
    assert r.props[3] == pytest.approx(0.0375 + 0.85 * 3 * 0.0375)
    r = Oracle.run(Oracle.build_graph(3, [0, 1], [1, 2]), SSSP, max_iterations=10)
    assert list(r.props) == [0.0, 1.0, 2.0]
    assert np.isinf(Oracle.run(Oracle.build_graph(3, [0], [1]), SSSP, max_iterations=10).props[2])
    assert Oracle.run(Oracle.dumbbell(2), SSSP, source=99, max_iterations=5).msg == \
        "sssp source vertex out of range"
    assert list(Oracle.run(Oracle.build_graph(4, [0, 1, 2, 3], [1, 0, 3, 2]), WCC,
                           max_iterations=10).props) == [0, 0, 2, 2]
    g = Oracle.power_law(200, 5.0, 2.2, 8)
    for budget in (1, 2, 5, 10):
        r = Oracle.run(g, BP, states=3, coupling=0.7, epsilon=1e-9, max_iterations=budget)
        assert np.all(np.abs(r.props.sum(axis=1) - 1.0) <= 1e-12)


def _dense_pagerank(g, d, iters):  # test_support.hpp:52-70
    n = g.n
    rank = np.full(n, 1.0 / n)
    dst = np.repeat(np.arange(n), np.diff(g.off.astype(np.int64)))
    for _ in range(iters):
        fresh = np.full(n, (1.0 - d) / n)
        np.add.at(fresh, dst, d * rank[g.src] / g.outdeg[g.src])
        rank = fresh
    return rank


def test_oracle_equivalence_dense_pagerank():  # acceptance criterion 2
    for seed in (1, 2, 3):
        g = Oracle.power_law(100, 5.0, 2.2, seed)
        r = Oracle.run(g, PR, max_iterations=300, epsilon=1e-16)
        assert np.abs(r.props - _dense_pagerank(g, 0.85, 300)).sum() < 1e-10


@pytest.mark.skipif(not Reference.available(), reason="reference build absent (no /root/reference)")
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_oracle_equals_live_reference(seed):
    g = Oracle.power_law(700, 7.0, 2.1, seed)
    gw = Oracle.random_graph(400, 5000, seed, True)
    u = Oracle.symmetrized(g)
    for scheme in (ACCURATE, SP, SMS, GG):
        kw = dict(scheme=scheme, sigma=0.45, theta=0.05, alpha=2, max_iterations=40, seed=seed)
        for graph, prog, pp in ((g, PR, {}), (gw, SSSP, dict(graded=True)), (u, WCC, {}),
                                (g, BP, {}), (g, BP, dict(states=4, coupling=0.6))):
            a = Oracle.run(graph, prog, **kw, **pp)
            b = Reference.run(graph, prog, **kw, **pp)
            assert a.status == b.status
            assert a.props.tobytes() == b.props.tobytes()
            assert (a.modes, a.processed_edges, a.active_vertices) == \
                (b.modes, b.processed_edges, b.active_vertices)


def test_metrics_known_answers():  # acceptance_main.cpp:322-370
    a1, e1 = [9, 8, 7, 1, 0], [9, 8, 1, 7, 0]
    assert Oracle.topk_error(a1, e1, 3) == 1.0 / 3.0
    v = [3, 1, 4, 1, 5]
    assert Oracle.topk_error(v, v, 2) == 0.0 and Oracle.topk_error(v, [1, 2, 3, 4, 5], 5) == 0.0
    assert Oracle.relative_error([7, 0, 0, 0], [0, 0, 0, 0]) == 0.25
    assert Oracle.relative_error([0] * 6 + [6] * 6, [0] * 12) == 0.5
    inf = float("inf")
    assert Oracle.stretch_error([0, 1, 2], [0, 1, 2]) == 0.0
    assert Oracle.stretch_error([0, inf], [0, 1]) == 1.0
    assert Oracle.stretch_error([0, 2, 2], [0, 1, 2]) == 0.25
    with pytest.raises(RuntimeError):
        Oracle.stretch_error([0, 1], [0, 2])


def test_oracle_sweep_matches_reference_golden_csv():  # test_bench.cpp:250-262
    from paper_2104_10039_b200 import sweep
    from tests.parity import oracle_runner
    import paper_2104_10039_b200 as ggb
    d = Oracle.dumbbell(4)
    plan = sweep.SweepPlan(algo="wcc", graph=ggb.Graph(d.n, d.off, d.src), graph_label="gen:dumbbell:4",
                           schemes=["sp", "gg"], sigma_grid=[0.4, 0.8], theta_grid=[0.5],
                           alpha_grid=[2], iterations=16, repeats=1, seeds=[1, 2])
    rows = sweep.run_sweep(plan, runner=oracle_runner)
    ours = sweep.mask_time_columns(sweep.emit_csv(rows, plan))
    with open(os.path.join(GOLDEN, "dumbbell4_sweep.csv")) as f:
        golden = sweep.mask_time_columns(f.read())
    assert ours == golden
