"""Shared parity helpers: run the same seeded case through the device engine
(paper_2104_10039_b200, via the C ABI) and the CPU oracle, and compare.

Bars (north_star): bit-exact for WCC labels and integer-weight SSSP
distances (and for every f64 SSSP, whose min-fold is exact); PR within
relative 1e-9; BP within 1e-6 (f64 beliefs) / 2e-6 (fp32 belief storage);
per-iteration modes, processed_edges and active_vertices identical; final
active-edge masks identical except edges whose influence lies within float
rounding of theta (counted and returned, never silently ignored).
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import BP, BP_EDGE, PR, SCHEMES, SSSP, WCC, Oracle

RTOL = {PR: 1e-9, BP: 1e-6, BP_EDGE: 2e-6}


class _OracleReport:
    def __init__(self, r):
        self.final_properties = r.props
        self.iterations_run = r.iterations_run
        self.total_processed_edges = r.total_processed_edges
        self.total_wall_seconds = 0.0
        self.per_iteration = r.processed_edges


def oracle_runner(graph, program, cfg):
    """runner(graph, program, EngineConfig) for paper_2104_10039_b200.sweep
    backed by the CPU oracle (tests only)."""
    import paper_2104_10039_b200 as ggb
    from oracle.oracle import CSC
    g = CSC(graph.n, graph.in_offsets, graph.in_sources,
            None if graph.weights is None else graph.weights.astype(np.float64), graph.out_degree)
    c = cfg.c()
    kw = dict(scheme=c.scheme, sigma=c.sigma, theta=c.theta, alpha=c.alpha,
              max_iterations=c.max_iterations, seed=c.seed, threads=max(c.threads, 1))
    if isinstance(program, ggb.PageRankProgram):
        r = Oracle.run(g, PR, damping=program.damping, epsilon=program.epsilon, **kw)
    elif isinstance(program, ggb.SsspProgram):
        r = Oracle.run(g, SSSP, source=program.source, graded=program.graded, **kw)
    elif isinstance(program, ggb.WccProgram):
        r = Oracle.run(g, WCC, **kw)
    elif isinstance(program, ggb.BeliefPropagationProgram):
        r = Oracle.run(g, BP, states=program.states, coupling=program.coupling,
                       epsilon=program.epsilon, **kw)
    else:
        raise TypeError(type(program))
    if r.status != 0:
        raise RuntimeError(r.msg)
    return _OracleReport(r)


def to_graph(ggb, g, weights=None):
    w = g.w if weights is None else weights
    return ggb.Graph(g.n, g.off, g.src, w, g.outdeg)


def device_program(ggb, prog, **pp):
    if prog == PR:
        return ggb.PageRankProgram(pp.get("damping", 0.85), pp.get("epsilon", 1e-7))
    if prog == SSSP:
        return ggb.SsspProgram(pp.get("source", 0), pp.get("graded", False))
    if prog == WCC:
        return ggb.WccProgram()
    if prog == BP:
        return ggb.BeliefPropagationProgram(pp.get("states", 2), pp.get("coupling", 0.8),
                                            pp.get("epsilon", 1e-6))
    if prog == BP_EDGE:
        return ggb.EdgeBeliefPropagationProgram(pp["prior_table"].reshape(-1, 2),
                                                pp.get("epsilon", 1e-6))
    raise ValueError(prog)


def compare(ggb, g, prog, scheme="accurate", sigma=1.0, theta=0.0, alpha=1, max_iterations=100,
            seed=0, dev_graph=None, device_weights=None, strict_counts=True, **pp):
    """Returns (device report, oracle result, mask mismatches)."""
    sch = SCHEMES[scheme]
    ref = Oracle.run(g, prog, scheme=sch, sigma=sigma, theta=theta, alpha=alpha,
                     max_iterations=max_iterations, seed=seed, want_flags=True, **pp)
    cfg = ggb.EngineConfig(scheme, sigma, theta, alpha, max_iterations, seed)
    graph = dev_graph if dev_graph is not None else to_graph(ggb, g, device_weights)
    program = device_program(ggb, prog, **pp)
    if ref.status == 2:
        try:
            ggb.run(graph, program, cfg)
        except ggb.EngineError as e:
            assert (e.iteration, e.vertex) == (ref.err_iteration, ref.err_vertex), (
                (e.iteration, e.vertex), (ref.err_iteration, ref.err_vertex))
            return None, ref, 0
        raise AssertionError(f"device run did not raise EngineError ({ref.msg})")
    assert ref.status == 0, ref.msg
    rep = ggb.run(graph, program, cfg, want_flags=True)
    mism = int(np.count_nonzero(rep.flags != ref.flags)) if g.e else 0
    if strict_counts:
        assert rep.iterations_run == ref.iterations_run, (rep.iterations_run, ref.iterations_run)
        assert [int(r.mode) for r in rep.per_iteration] == ref.modes
        assert [r.processed_edges for r in rep.per_iteration] == ref.processed_edges
        assert [r.active_vertices for r in rep.per_iteration] == ref.active_vertices
        assert rep.total_processed_edges == ref.total_processed_edges
    props, rprops = rep.final_properties, ref.props
    if prog in (SSSP, WCC):
        assert np.array_equal(props, rprops), "exact program differs"
    else:
        np.testing.assert_allclose(props, rprops, rtol=RTOL[prog], atol=1e-300)
    return rep, ref, mism
