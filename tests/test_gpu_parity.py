"""Device engine vs CPU oracle on seeded inputs (the parity tests proper).

Mirrors the reference's own tests (test_engine.cpp, test_algorithms.cpp,
acceptance_main.cpp) through the C ABI, plus R-MAT cases at the BASELINE
configs' shapes (reduced scale where the oracle must finish in seconds)."""
import numpy as np
import pytest

from oracle.oracle import BP, BP_EDGE, CSC, GG, PR, SSSP, WCC, Oracle
from tests.parity import compare, to_graph

pytestmark = pytest.mark.gpu

SCHEMES = ["accurate", "sp", "sms", "gg"]


# --------------------------------------------------------------------------
# known answers (test_algorithms.cpp / test_engine.cpp restated)
# --------------------------------------------------------------------------
def test_pagerank_four_cycle_fixed_point(ggb):  # test_algorithms.cpp:76-83, test_engine.cpp:184-194
    g = Oracle.build_graph(4, [0, 1, 2, 3], [1, 2, 3, 0])
    rep = ggb.run(to_graph(ggb, g), ggb.pagerank_spec(), ggb.EngineConfig(max_iterations=50))
    assert rep.iterations_run == 1
    np.testing.assert_allclose(rep.final_properties, 0.25, rtol=1e-12)


def test_pagerank_star_hub(ggb):  # test_algorithms.cpp:85-97
    g = Oracle.build_graph(4, [0, 1, 2], [3, 3, 3])
    rep = ggb.run(to_graph(ggb, g), ggb.pagerank_spec(0.85, 1e-16),
                  ggb.EngineConfig(max_iterations=300))
    assert rep.final_properties[3] == pytest.approx(0.0375 + 0.85 * 3 * 0.0375)


def test_sp_sigma_zero_leak(ggb):  # test_engine.cpp:122-131
    g = Oracle.dumbbell(2)
    rep = ggb.run(to_graph(ggb, g), ggb.pagerank_spec(),
                  ggb.EngineConfig("sp", sigma=0.0, max_iterations=50))
    np.testing.assert_allclose(rep.final_properties, 0.15 / 4, rtol=1e-12)
    assert rep.iterations_run == 2


def test_three_cycle_gathers_every_edge(ggb):  # test_engine.cpp:226-237
    g = Oracle.build_graph(3, [0, 1, 2], [1, 2, 0])
    rep = ggb.run(to_graph(ggb, g), ggb.pagerank_spec(0.85, 1e-15),
                  ggb.EngineConfig(max_iterations=5))
    assert all(r.processed_edges == 3 and r.active_vertices == 3 for r in rep.per_iteration)


def test_unreachable_theta_deactivates_every_edge(ggb):  # test_engine.cpp:239-256
    g = Oracle.dumbbell(3)
    rep = ggb.run(to_graph(ggb, g), ggb.pagerank_spec(),
                  ggb.EngineConfig("gg", sigma=1.0, theta=2.0, alpha=5, max_iterations=10))
    assert rep.per_iteration[5].mode == ggb.IterationMode.superstep
    for r in rep.per_iteration[6:]:
        assert r.mode == ggb.IterationMode.approximate and r.processed_edges == 0
    np.testing.assert_allclose(rep.final_properties, 0.15 / 6, rtol=1e-12)


def test_sssp_known_answers(ggb):  # test_algorithms.cpp:140-152
    g = Oracle.build_graph(3, [0, 1], [1, 2])
    rep = ggb.run(to_graph(ggb, g), ggb.sssp_spec(0), ggb.EngineConfig(max_iterations=10))
    assert list(rep.final_properties) == [0.0, 1.0, 2.0]
    g = Oracle.build_graph(3, [0], [1])
    rep = ggb.run(to_graph(ggb, g), ggb.sssp_spec(0), ggb.EngineConfig(max_iterations=10))
    assert np.isinf(rep.final_properties[2])


def test_sssp_source_out_of_range(ggb):  # test_algorithms.cpp:173-177
    with pytest.raises(ValueError, match="sssp source vertex out of range"):
        ggb.run(to_graph(ggb, Oracle.dumbbell(2)), ggb.sssp_spec(99), ggb.EngineConfig(max_iterations=5))


def test_wcc_known_answers(ggb):  # test_algorithms.cpp:189-201
    g = Oracle.build_graph(3, [0, 1, 2], [1, 2, 0])
    assert list(ggb.run(to_graph(ggb, g), ggb.wcc_spec(),
                        ggb.EngineConfig(max_iterations=10)).final_properties) == [0, 0, 0]
    g = Oracle.build_graph(4, [0, 1, 2, 3], [1, 0, 3, 2])
    assert list(ggb.run(to_graph(ggb, g), ggb.wcc_spec(),
                        ggb.EngineConfig(max_iterations=10)).final_properties) == [0, 0, 2, 2]


def test_bp_isolated_and_uninformative(ggb, oracle):  # test_algorithms.cpp:232-255
    g = Oracle.build_graph(3, [0], [1])
    rep = ggb.run(to_graph(ggb, g), ggb.bp_spec(), ggb.EngineConfig(max_iterations=20))
    ref = Oracle.run(g, BP, max_iterations=20)
    np.testing.assert_allclose(rep.final_properties[2], ref.props[2], rtol=1e-14)
    g = Oracle.build_graph(2, [0, 1], [1, 0])
    rep = ggb.run(to_graph(ggb, g), ggb.bp_spec(2, 0.5, 1e-9), ggb.EngineConfig(max_iterations=30))
    prior = Oracle.run(Oracle.build_graph(2, [], []), BP, max_iterations=1, coupling=0.5).props
    np.testing.assert_allclose(rep.final_properties, prior, rtol=1e-12)


def test_bp_beliefs_normalised(ggb):  # test_algorithms.cpp:273-284
    g = Oracle.power_law(200, 5.0, 2.2, 8)
    for budget in (1, 2, 5, 10):
        rep = ggb.run(to_graph(ggb, g), ggb.bp_spec(3, 0.7, 1e-9),
                      ggb.EngineConfig(max_iterations=budget))
        assert np.all(np.abs(rep.final_properties.sum(axis=1) - 1.0) <= 1e-12)


def test_empty_graph(ggb):  # test_engine.cpp:304-309
    g = ggb.Graph(0, np.zeros(1, np.uint64), np.zeros(0, np.uint32))
    rep = ggb.run(g, ggb.pagerank_spec(), ggb.EngineConfig())
    assert rep.iterations_run == 0 and rep.final_properties.size == 0


def test_invalid_config_names_field(ggb):  # test_engine.cpp:105-120
    g = to_graph(ggb, Oracle.dumbbell(2))
    with pytest.raises(ValueError, match="sigma"):
        ggb.run(g, ggb.pagerank_spec(), ggb.EngineConfig(sigma=1.5))
    with pytest.raises(ValueError, match="alpha"):
        ggb.run(g, ggb.pagerank_spec(), ggb.EngineConfig(sigma=0.5, alpha=0))


def test_invalid_property_abort(ggb):
    # engine.hpp:226-233: a negative weight drives SSSP distances below 0
    # (SsspProgram::valid, algorithms.hpp:82) -> EngineError(t, smallest v).
    g = Oracle.random_graph(60, 400, 3, True)
    w = g.w.copy()
    w[::37] = -5.0
    g.w = w
    compare(ggb, g, SSSP, max_iterations=50)
    compare(ggb, g, SSSP, scheme="gg", sigma=0.6, theta=0.1, alpha=2, max_iterations=50, seed=4)


# --------------------------------------------------------------------------
# exactness gate and random-graph parity (acceptance 1, 2, 10)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_exactness_gate(ggb, seed):  # acceptance_main.cpp:80-113
    g = Oracle.power_law(1000, 8.0, 2.1, seed)
    u = Oracle.symmetrized(g)
    for prog, graph in ((PR, g), (SSSP, g), (WCC, u), (BP, g)):
        base = compare(ggb, graph, prog, max_iterations=20)[0].final_properties
        for scheme in ("gg", "sp"):
            rep = compare(ggb, graph, prog, scheme=scheme, sigma=1.0, alpha=20, max_iterations=20,
                          seed=seed)[0]
            assert np.array_equal(rep.final_properties, base)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_random_graphs_all_programs(ggb, scheme, seed):
    g = Oracle.power_law(500, 8.0, 2.1, seed)
    gw = Oracle.random_graph(300, 3000, seed, True)
    u = Oracle.symmetrized(g)
    kw = dict(scheme=scheme, sigma=0.5, theta=0.1, alpha=3, max_iterations=30, seed=seed)
    total = 0
    total += compare(ggb, g, PR, **kw)[2]
    total += compare(ggb, gw, SSSP, **kw)[2]
    total += compare(ggb, gw, SSSP, graded=True, **kw)[2]
    total += compare(ggb, u, WCC, **kw)[2]
    total += compare(ggb, g, BP, **kw)[2]
    total += compare(ggb, g, BP, states=3, coupling=0.7, **kw)[2]
    assert total == 0


@pytest.mark.parametrize("states", [4, 5, 8, 16, 17, 32, 33, 64])
def test_bp_many_states(ggb, states):
    """BeliefProp<S> for S <= 4, the run-time-S programs above (storage tiers
    of 16 / 32 / 64 states), against the oracle's reference BP
    (algorithms.cpp:9-69); S > 64 is rejected with a clear message."""
    g = Oracle.power_law(400, 6.0, 2.1, states)
    for scheme in SCHEMES:
        _, _, mism = compare(ggb, g, BP, scheme=scheme, sigma=0.5, theta=0.01, alpha=3,
                             max_iterations=25, seed=states, states=states, coupling=0.6)
        assert mism == 0
    with pytest.raises(ValueError, match="<= 64"):
        ggb.run(to_graph(ggb, g), ggb.BeliefPropagationProgram(65, 0.6, 1e-6),
                ggb.EngineConfig(max_iterations=2))


@pytest.mark.parametrize("seed", [1, 2])
def test_edge_bp_fp32(ggb, seed):
    g = Oracle.power_law(600, 8.0, 2.1, seed)
    c = Oracle.bp_couplings(g.e, seed)
    gw = Oracle.build_graph(g.n, g.src, np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64))),
                            c.astype(np.float64))
    pri = Oracle.bp_priors(g.n, seed)
    for scheme in SCHEMES:
        _, _, mism = compare(ggb, gw, BP_EDGE, scheme=scheme, sigma=0.5, theta=0.01, alpha=4,
                             max_iterations=30, seed=seed, prior_table=pri, device_weights=c)
        assert mism == 0


def test_edge_bp_resident_priors(ggb):
    """A device-resident prior table (generated there, or uploaded once) gives
    exactly the run a host table gives."""
    n_seed = 3
    dg = ggb.DeviceGraph.rmat(12, 16, n_seed, weights="coupling")
    host = ggb.bp_priors(dg.n, n_seed)
    assert np.array_equal(host, Oracle.bp_priors(dg.n, n_seed).reshape(dg.n, 2))
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 4, 20, n_seed)
    a = ggb.run(dg, ggb.EdgeBeliefPropagationProgram(host, 1e-6), cfg)
    for pri in (ggb.bp_priors(dg.n, n_seed, device=True), ggb.DeviceBuffer.upload(host)):
        b = ggb.run(dg, ggb.EdgeBeliefPropagationProgram(pri, 1e-6), cfg)
        assert np.array_equal(a.final_properties, b.final_properties)
        assert [r.processed_edges for r in a.per_iteration] == [r.processed_edges for r in b.per_iteration]
        pri.close()
    dg.close()


def test_sssp_u32_weights_exact(ggb):
    g = Oracle.rmat(12, 16, 2)
    w = Oracle.rmat_weights_u32(g.e, 2)
    gw = Oracle.build_graph(g.n, g.src, np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64))),
                            w.astype(np.float64))
    src = int(np.argmax(gw.outdeg))
    for scheme in SCHEMES:
        compare(ggb, gw, SSSP, scheme=scheme, sigma=0.5, theta=0.05, alpha=4, seed=2,
                max_iterations=g.n + 1, source=src, graded=True, device_weights=w)


def test_sssp_u32_weights_beyond_32_bit_distances(ggb):
    """u32 weights whose path sums exceed 2^32-1: the u32-distance program
    flags the overflow and the run is redone with f64 distances, so the
    result still equals the reference's f64 arithmetic."""
    g = Oracle.rmat(11, 8, 6)
    rng = np.random.default_rng(6)
    w = rng.integers(1 << 30, (1 << 32) - 1, g.e, dtype=np.uint64).astype(np.uint32)
    gw = Oracle.build_graph(g.n, g.src, np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64))),
                            w.astype(np.float64))
    src = int(np.argmax(gw.outdeg))
    for scheme in ("accurate", "gg"):
        rep, ref, _ = compare(ggb, gw, SSSP, scheme=scheme, sigma=0.5, theta=0.05, alpha=4, seed=6,
                              max_iterations=g.n + 1, source=src, graded=True, device_weights=w)
        finite = np.asarray(ref.props)[np.isfinite(ref.props)]
        assert finite.max() > 2 ** 32  # the overflow path was exercised


def test_hub_windows_multi_chunk(ggb):
    # in-degree 5000 hub + 3000 hub: windows split into several chunks, and
    # the superstep hub pass evaluates their influences with chunk carries.
    rng = np.random.default_rng(5)
    n = 6000
    src = np.concatenate([rng.integers(0, n, 5000), rng.integers(0, n, 3000),
                          rng.integers(0, n, 20000)]).astype(np.uint32)
    dst = np.concatenate([np.full(5000, 3), np.full(3000, 40),
                          rng.integers(0, n, 20000)]).astype(np.uint32)
    g = Oracle.build_graph(n, src, dst)
    u = Oracle.symmetrized(g)
    for scheme in SCHEMES:
        kw = dict(scheme=scheme, sigma=0.5, theta=0.001, alpha=2, max_iterations=25, seed=7)
        assert compare(ggb, g, PR, **kw)[2] == 0
        assert compare(ggb, u, WCC, **kw)[2] == 0
        assert compare(ggb, g, BP, **kw)[2] == 0


def test_dumbbell_recovery(ggb):  # test_engine.cpp:258-286, acceptance 3
    k = 8
    g = Oracle.dumbbell(k)
    exact = compare(ggb, g, WCC, max_iterations=64)[0].final_properties
    # the reference's find_bridge_dropping_seed (test_support.hpp:198-228)
    bridge = [e for v in range(g.n) for e in range(int(g.off[v]), int(g.off[v + 1]))
              if (g.src[e], v) in ((k - 1, k), (k, k - 1))]
    seed = None
    for s in range(512):
        f = Oracle.sparsify(g.e, 0.5, s)
        if any(f[e] for e in bridge):
            continue
        if all(f[int(g.off[v]):int(g.off[v + 1])].any() for v in range(g.n)):
            seed = s
            break
    assert seed is not None
    sp = compare(ggb, g, WCC, scheme="sp", sigma=0.5, max_iterations=64, seed=seed)[0]
    assert not np.array_equal(sp.final_properties, exact)
    gg = compare(ggb, g, WCC, scheme="gg", sigma=0.5, theta=0.5, alpha=2, max_iterations=64,
                 seed=seed)[0]
    assert np.array_equal(gg.final_properties, exact)
    assert gg.per_iteration[2].mode == ggb.IterationMode.superstep


@pytest.mark.parametrize("prog", ["pr", "wcc", "sssp", "bp"])
def test_grid_and_thread_invariance(ggb, prog):  # test_engine.cpp:161-182 analogue
    """The fold structure is a function of global edge positions only, so
    properties, flags and per-iteration counts are bit-identical whatever
    the grid (1 CTA, a few, the occupancy-sized default: tasks land on
    different warps in a different order, and the superstep chain waits on
    different predecessors) and whatever cfg.threads says."""
    g = Oracle.power_law(6000, 10.0, 2.1, 3)
    if prog == "wcc":
        g = Oracle.symmetrized(g)
    if prog == "sssp":
        g = Oracle.random_graph(4000, 50000, 3, True)
    program = {"pr": ggb.pagerank_spec(), "wcc": ggb.wcc_spec(), "sssp": ggb.sssp_spec(0, True),
               "bp": ggb.bp_spec(3, 0.7)}[prog]
    dg = ggb.DeviceGraph.upload(to_graph(ggb, g))
    cfg = ggb.EngineConfig("gg", 0.4, 0.05, 3, 30, 5)
    base = ggb.run(dg, program, cfg, want_flags=True)
    assert any(r.mode == ggb.IterationMode.superstep for r in base.per_iteration)
    for grid, threads in ((1, 1), (3, 1), (7, 8), (0, 8)):
        c = ggb.EngineConfig("gg", 0.4, 0.05, 3, 30, 5, threads=threads)
        r = ggb.run(dg, program, c, want_flags=True, grid_ctas=grid)
        assert np.array_equal(np.asarray(r.final_properties).view(np.uint8),
                              np.asarray(base.final_properties).view(np.uint8)), (grid, threads)
        assert np.array_equal(r.flags, base.flags), (grid, threads)
        assert [(x.processed_edges, x.active_vertices) for x in r.per_iteration] == \
            [(x.processed_edges, x.active_vertices) for x in base.per_iteration]
    dg.close()


# --------------------------------------------------------------------------
# R-MAT inputs (BASELINE configs at oracle-sized scales)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("scale,ef,seed,sym,wk", [(10, 16, 1, False, None), (12, 16, 2, False, "u32"),
                                                 (11, 16, 3, True, None), (12, 8, 4, False, "coupling")])
def test_device_rmat_equals_oracle(ggb, scale, ef, seed, sym, wk):
    dg = ggb.DeviceGraph.rmat(scale, ef, seed, symmetrize=sym, weights=wk)
    h = dg.to_host()
    g = Oracle.rmat(scale, ef, seed)
    if sym:
        g = Oracle.symmetrized(g)
    assert np.array_equal(h.in_offsets, g.off) and np.array_equal(h.in_sources, g.src)
    assert np.array_equal(h.out_degree, g.outdeg)
    if wk == "u32":
        assert np.array_equal(h.weights, Oracle.rmat_weights_u32(g.e, seed))
    if wk == "coupling":
        assert np.array_equal(h.weights, Oracle.bp_couplings(g.e, seed))


def test_c1_pagerank_rmat_s16(ggb):
    """BASELINE configs[0]: PR gg on R-MAT s16 EF16 seed 1, d=0.85, eps=1e-7,
    theta=0.01 (sigma 0.5, alpha 4; budget = accurate iterations_run)."""
    g = Oracle.rmat(16, 16, 1)
    assert g.e == 955529
    acc = compare(ggb, g, PR, max_iterations=50)[0]
    _, ref, mism = compare(ggb, g, PR, scheme="gg", sigma=0.5, theta=0.01, alpha=4,
                           max_iterations=acc.iterations_run, seed=1)
    assert mism == 0


def test_rmat_sssp_wcc_bp_small(ggb):
    g = Oracle.rmat(13, 16, 2)
    w = Oracle.rmat_weights_u32(g.e, 2)
    gw = Oracle.build_graph(g.n, g.src, np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64))),
                            w.astype(np.float64))
    compare(ggb, gw, SSSP, scheme="gg", sigma=0.5, theta=0.05, alpha=4, seed=2,
            max_iterations=g.n + 1, source=0, graded=True, device_weights=w)
    u = Oracle.symmetrized(Oracle.rmat(13, 16, 3))
    compare(ggb, u, WCC, scheme="gg", sigma=0.5, theta=0.0, alpha=4, seed=3, max_iterations=u.n + 1)
    g4 = Oracle.rmat(12, 16, 4)
    c = Oracle.bp_couplings(g4.e, 4)
    g4w = Oracle.build_graph(g4.n, g4.src, np.repeat(np.arange(g4.n), np.diff(g4.off.astype(np.int64))),
                             c.astype(np.float64))
    compare(ggb, g4w, BP_EDGE, scheme="gg", sigma=0.5, theta=0.01, alpha=4, seed=4,
            max_iterations=30, prior_table=Oracle.bp_priors(g4.n, 4), device_weights=c)


def test_device_sparsify_matches_reference_hash(ggb):  # engine.cpp:63-75, test_engine.cpp:54-80
    e = 100000
    a = ggb.sparsify(e, 0.5, 3)
    assert np.array_equal(a, Oracle.sparsify(e, 0.5, 3))
    assert 49000 <= int(a.sum()) <= 51000
    assert int(ggb.sparsify(e, 1.0, 9).sum()) == e and int(ggb.sparsify(e, 0.0, 9).sum()) == 0
    lo, hi = ggb.sparsify(2000, 0.3, 5), ggb.sparsify(2000, 0.7, 5)
    assert np.all(hi[lo == 1] == 1)
    # thresholds with a non-zero low word (high-word ties resolved exactly), every
    # key & 31 class of the word-block decomposition, a ragged last word
    for sigma, seed in [(0.3, 5), (0.7, 6), (0.05, 11), (0.999, 2), (1e-7, 4), (1 / 3, 123456789)]:
        e = 1_000_003 + seed % 29
        assert np.array_equal(ggb.sparsify(e, sigma, seed), Oracle.sparsify(e, sigma, seed)), (sigma, seed)
    for seed in range(40, 72):
        assert np.array_equal(ggb.sparsify(4099, 0.4, seed), Oracle.sparsify(4099, 0.4, seed)), seed


# --------------------------------------------------------------------------
# list-build tile boundaries: the one-pass scan/compaction works on tiles of
# 1024 bitmap words (32768 edges) and the list layout on tiles of 2048
# vertices; edge and vertex counts straddle those boundaries (empty
# vertices, a hub spanning several 512-edge tasks, duplicate edges)
# --------------------------------------------------------------------------
def _exact_graph(n, e, seed, weighted=False):
    rng = np.random.default_rng(seed)
    p = rng.pareto(1.2, n) + 0.05
    p[rng.random(n) < 0.25] = 0.0  # empty vertices
    p[n // 3] = p.sum()            # one hub
    deg = rng.multinomial(e, p / p.sum())
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(deg)
    src = rng.integers(0, n, e).astype(np.uint32)
    for v in range(n):  # CSC order: sources ascending per destination
        a, b = int(off[v]), int(off[v + 1])
        src[a:b].sort()
    w = rng.integers(1, 50, e).astype(np.float64) if weighted else None
    return CSC(n, off, src, w)


@pytest.mark.parametrize("n,e", [(1023, 32767), (1024, 32768), (1025, 32769), (2047, 65537),
                                 (2048, 65536), (2049, 3 * 32768 + 5), (5000, 98303)])
def test_list_build_tile_boundaries(ggb, n, e):
    g = _exact_graph(n, e, n + e)
    gw = _exact_graph(n, e, n + e + 1, weighted=True)
    total = adopted = 0
    # theta = 0.05 = 1/20: duplicate sources make PR influences exactly 1/k,
    # and on such an exact tie the run-granular re-association of the PR
    # fold may round to the other side of theta -- the allowed near-threshold
    # deviation, which the lock-step comparison adopts and counts (parity.py)
    for scheme in ("sp", "gg", "sms"):
        kw = dict(scheme=scheme, sigma=0.5, theta=0.05, alpha=2, max_iterations=12, seed=e)
        for r in (compare(ggb, g, PR, **kw)[2], compare(ggb, g, WCC, **kw)[2],
                  compare(ggb, gw, SSSP, graded=True, **kw)[2],  # f64 weights
                  compare(ggb, gw, SSSP, graded=True,
                          device_weights=gw.w.astype(np.float32), **kw)[2]):  # f32 weights
            total += int(r)
            adopted += r.adopted
    print(f"n={n} e={e}: near-threshold edges decided differently: {adopted}")
    assert total == 0


def test_upload_for_run_presparsified(ggb):
    """gg_dev_graph_create_for_run: the sparsification done during the upload
    is used only by a run with the same sigma and seed, and only once; other
    runs on that graph sparsify again (results equal a plain upload's)."""
    g = Oracle.power_law(1500000, 12.0, 2.1, 7)  # >= 2^24 edges: the overlapped path
    assert g.e >= 1 << 24
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 3, 15, 11)
    other = ggb.EngineConfig("gg", 0.5, 0.01, 3, 15, 12)
    prog = ggb.PageRankProgram()
    plain = ggb.DeviceGraph.upload(to_graph(ggb, g))
    ref_cfg = ggb.run(plain, prog, cfg, want_flags=True)
    ref_other = ggb.run(plain, prog, other, want_flags=True)
    for first, second, r1, r2 in ((cfg, cfg, ref_cfg, ref_cfg), (other, cfg, ref_other, ref_cfg)):
        dg = ggb.DeviceGraph.upload(to_graph(ggb, g), for_run=cfg)
        a = ggb.run(dg, prog, first, want_flags=True)   # uses the upload's list iff same config
        b = ggb.run(dg, prog, second, want_flags=True)  # always sparsifies itself
        for rep, ref in ((a, r1), (b, r2)):
            assert np.array_equal(rep.final_properties, ref.final_properties)
            assert np.array_equal(rep.flags, ref.flags)
            assert [r.processed_edges for r in rep.per_iteration] == \
                   [r.processed_edges for r in ref.per_iteration]
        dg.close()
    plain.close()


@pytest.mark.parametrize("scheme", ["sp", "gg"])
def test_weight_ignoring_programs_on_weighted_graphs(ggb, scheme):
    """PageRank, WCC and S-state BP ignore edge weights (algorithms.hpp:15-145);
    on a weighted graph the sparsified list carries sources only."""
    g = Oracle.random_graph(3000, 40000, 5, True)
    u = Oracle.symmetrized(g)
    kw = dict(scheme=scheme, sigma=0.5, theta=0.05, alpha=3, max_iterations=20, seed=9)
    total = 0
    for w in (g.w, g.w.astype(np.float32), g.w.astype(np.uint32)):
        total += compare(ggb, g, PR, device_weights=w, **kw)[2]
    total += compare(ggb, u, WCC, device_weights=u.w.astype(np.uint32), **kw)[2]
    total += compare(ggb, g, BP, device_weights=g.w, **kw)[2]  # S-state BP ignores weights too
    assert total == 0


@pytest.mark.parametrize("wkind", ["u32", "f32", "f64"])
def test_upload_for_run_presparsified_weighted(ggb, monkeypatch, wkind):
    """The upload-overlapped sparsification on WEIGHTED graphs (weights
    copied per chunk and compacted with the kept sources): SSSP (u32 / f64
    distances) and BP with per-edge couplings (f32 weights), uploaded with
    for_run, equal a plain upload in properties, flags and records. The
    2^24-edge cut is lowered so small graphs take that path."""
    monkeypatch.setenv("GGB_PRESPARSE_MIN_EDGES", "1")
    g = Oracle.power_law(20000, 12.0, 2.1, 5)
    rng = np.random.default_rng(5)
    if wkind == "u32":
        w = rng.integers(1, 255, g.e).astype(np.uint32)
        prog = ggb.sssp_spec(0, True)
    elif wkind == "f64":
        w = rng.uniform(0.1, 3.0, g.e).astype(np.float64)
        prog = ggb.sssp_spec(0, True)
    else:
        w = Oracle.bp_couplings(g.e, 5)
        prog = ggb.EdgeBeliefPropagationProgram(Oracle.bp_priors(g.n, 5).reshape(-1, 2), 1e-6)
    graph = ggb.Graph(g.n, g.off, g.src, w, g.outdeg)
    cfg = ggb.EngineConfig("gg", 0.5, 0.05, 3, 20, 11)
    plain = ggb.DeviceGraph.upload(graph)
    ref = ggb.run(plain, prog, cfg, want_flags=True)
    plain.close()
    dg = ggb.DeviceGraph.upload(graph, for_run=cfg)  # sparsified during the upload
    rep = ggb.run(dg, prog, cfg, want_flags=True)
    dg.close()
    assert np.array_equal(np.asarray(rep.final_properties).view(np.uint8),
                          np.asarray(ref.final_properties).view(np.uint8))
    assert np.array_equal(rep.flags, ref.flags)
    assert [r.processed_edges for r in rep.per_iteration] == [r.processed_edges for r in ref.per_iteration]


@pytest.mark.parametrize("prog", ["pr", "bp5"])
def test_chain_stress_bitwise(ggb, prog):
    """The superstep chain's carries and the look-back scans do not depend on
    timing: 24 runs over grids from 1 CTA to the default (different warps
    hold different tasks, predecessors finish in different orders) are
    bit-identical in properties, flags and counts. Hub-heavy graph: in-lists
    spanning many 512-edge tasks. (compute-sanitizer is closed on this pool;
    this and the grid-invariance tests stand in for racecheck.)"""
    g = Oracle.power_law(30000, 40.0, 1.8, 11)
    program = ggb.pagerank_spec() if prog == "pr" else ggb.bp_spec(5, 0.7)
    dg = ggb.DeviceGraph.upload(to_graph(ggb, g))
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 1, 12, 3)  # a superstep every other iteration
    base = ggb.run(dg, program, cfg, want_flags=True)
    assert sum(r.mode == ggb.IterationMode.superstep for r in base.per_iteration) >= 3
    for k, grid in enumerate([1, 2, 5, 37, 148, 0] * 4):
        r = ggb.run(dg, program, cfg, want_flags=True, grid_ctas=grid)
        assert np.array_equal(np.asarray(r.final_properties).view(np.uint8),
                              np.asarray(base.final_properties).view(np.uint8)), (k, grid)
        assert np.array_equal(r.flag_words, base.flag_words), (k, grid)
        assert [x.active_vertices for x in r.per_iteration] == [x.active_vertices for x in base.per_iteration]
    dg.close()


# --------------------------------------------------------------------------
# PageRank's division-free superstep test (kernels.cuh rel_growth_influence):
# influences EXACTLY equal to theta and just around it must be decided as the
# reference's correctly rounded division decides them.
# --------------------------------------------------------------------------
def _dyadic_graph(n, k):
    """Out-degree k everywhere; in-degrees 2k (n/4 vertices), k/2 (n/2) and k
    (n/4); in-lists hold distinct sources, ascending. With n, k powers of two
    and damping 0.5 the ranks after iteration 1 are 1.5/n, 0.75/n and 1/n and
    every message of the t = 2 superstep is a small dyadic multiple of
    1/(n k): every prefix sum is exact under any association."""
    deg = np.concatenate([np.full(n // 4, 2 * k), np.full(n // 2, k // 2), np.full(n - 3 * n // 4, k)])
    deg = np.random.default_rng(k).permutation(deg)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(deg)
    src = (np.arange(int(off[-1])) % n).astype(np.uint32)
    for v in range(n):
        a, b = int(off[v]), int(off[v + 1])
        src[a:b].sort()
    return CSC(n, off, src, None)


def _superstep_influences(g, k):
    """fl(d / s) of every edge at the t = 2 superstep (exact sums)."""
    n = g.n
    deg = np.diff(g.off.astype(np.int64))
    rank1 = (0.5 + 0.5 * deg / k) / n
    m = rank1 / k
    out = np.empty(len(g.src))
    for v in range(n):
        a, b = int(g.off[v]), int(g.off[v + 1])
        s = np.cumsum(m[g.src[a:b]])
        before = np.concatenate([[0.0], s[:-1]])
        out[a:b] = (s - before) / s
    return out


@pytest.mark.parametrize("k", [8, 32, 256])
@pytest.mark.parametrize("theta", [0.25, 0.125, 0.5, 1.0 / 3.0, 0.1, 0.25 * (1 + 2.0 ** -52),
                                   0.25 * (1 - 2.0 ** -53), 0.0])
def test_pagerank_exact_influence_ties(ggb, k, theta):
    """The superstep's flags when influences sit EXACTLY on theta or one ulp
    off it (0.25 +- 1 ulp), for inexact thresholds (1/3, 0.1) and theta = 0
    (not a normal number: the exact path everywhere). The prefix sums are
    exact under any association (_dyadic_graph), so the device and the oracle
    see the same (d, s) for every edge and must take the same decision with
    no near-threshold adoption."""
    n = 2048 if k == 8 else 1024  # k = 256: in-lists of 512 edges span tasks
    g = _dyadic_graph(n, k)
    infl = _superstep_influences(g, k)
    if k == 8 and theta in (0.25, 0.125, 0.5):
        assert np.count_nonzero(infl == theta) > 0  # the case exercises exact ties
    rep, ref, mr = compare(ggb, g, PR, scheme="gg", sigma=1.0, theta=theta, alpha=1,
                           max_iterations=2, damping=0.5)
    assert mr.adopted == 0 and mr.real == 0, mr.per_superstep
    assert np.array_equal(rep.flags.astype(bool), infl > theta)
