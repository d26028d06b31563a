"""Shared parity helpers: run the same seeded case through the device engine
(paper_2104_10039_b200, via the C ABI) and the CPU oracle, and compare.

Bars (north_star): bit-exact for WCC labels and integer-weight SSSP
distances (and for every f64 SSSP, whose min-fold is exact); PR within
relative 1e-9; BP within 1e-6 (f64 beliefs) / 2e-6 (fp32 belief storage);
per-iteration modes, processed_edges and active_vertices identical; final
active-edge masks identical except edges whose influence lies within float
rounding of theta, which are counted and returned.

Mask parity is checked in LOCK-STEP (oracle og_run_ex): the device's flags
right after every superstep are compared edge by edge with the oracle's
own estatus decision. A differing edge whose oracle influence lies inside
the program's rounding band of theta (NEAR_UNIT below; the band formula is
in oracle/gg_oracle.h) is a near-threshold edge: the oracle adopts the
device's decision for it, so the rest of the run is compared on the same
flag set. A differing edge outside the band is a REAL mismatch and fails
the test. Every comparison reports how many near-threshold edges there were.
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import BP, BP_EDGE, PR, SCHEMES, SSSP, WCC, Oracle

RTOL = {PR: 1e-9, BP: 1e-6, BP_EDGE: 2e-6}

# Near-threshold band unit per program (oracle/gg_oracle.h og_lockstep):
# band = unit * ((k + 4) * max(infl, theta) + 4), k = the edge's position
# in its in-list. The device re-associates the prefix accumulator (16-edge
# runs joined by `combine`): f64 sums move an influence by at
# most ~(k + 2) * 2^-53 relative plus ~2^-53 absolute; the unit carries a
# safety factor 8 (PR) / 64 (BP: a renormalised product per edge). fp32-
# stored BP (C4) messages can differ by one fp32 ulp (2^-24) where an f64
# re-association difference crosses an fp32 rounding boundary: unit 2^-22.
# The min programs (SSSP, WCC) fold exactly under any grouping: unit 0, so
# any differing flag is a real mismatch.
NEAR_UNIT = {PR: 2.0 ** -50, BP: 2.0 ** -47, BP_EDGE: 2.0 ** -22, SSSP: 0.0, WCC: 0.0}


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


def superstep_flags(ggb, graph, program, cfg, rep):
    """The device's flag bitmap right after each superstep of `rep` (a run
    capped at that iteration ends with it; the engine is deterministic)."""
    import paper_2104_10039_b200 as m
    out = []
    its = [i + 1 for i, r in enumerate(rep.per_iteration) if r.mode == m.IterationMode.superstep]
    for t in its:
        if t == rep.iterations_run and rep.flag_words is not None:
            out.append(rep.flag_words)
            continue
        c = m.EngineConfig(cfg.scheme, cfg.sigma, cfg.theta, cfg.alpha, t, cfg.seed, cfg.threads)
        out.append(ggb.run(graph, program, c, want_flags=True, device_output=True).flag_words)
    return out


class MaskReport(int):
    """Final-mask mismatches (an int, 0 when parity holds) carrying the
    lock-step counts: near (edges in the band), adopted (near-threshold
    edges the device decided the other way), real (mismatches outside)."""
    near = adopted = real = 0
    per_superstep: list = []


def lockstep(ggb, g, prog, graph, program, cfg, rep, threads=1, **pp):
    """Oracle run in lock-step with the device report `rep`; returns
    (oracle result, MaskReport)."""
    dev = superstep_flags(ggb, graph, program, cfg, rep)
    c = cfg.c()
    ref = Oracle.run(g, prog, scheme=c.scheme, sigma=c.sigma, theta=c.theta, alpha=c.alpha,
                     max_iterations=c.max_iterations, seed=c.seed, threads=threads,
                     want_flags=rep.flags is not None, device_flags=dev,
                     tol_unit=NEAR_UNIT[prog], **pp)
    assert ref.status == 0, ref.msg
    mism = int(np.count_nonzero(rep.flags != ref.flags)) if (g.e and rep.flags is not None) else 0
    mr = MaskReport(mism)
    mr.per_superstep = ref.lockstep
    mr.near = sum(s["near"] for s in ref.lockstep)
    mr.adopted = sum(s["adopted"] for s in ref.lockstep)
    mr.real = sum(s["real"] for s in ref.lockstep)
    return ref, mr


def compare(ggb, g, prog, scheme="accurate", sigma=1.0, theta=0.0, alpha=1, max_iterations=100,
            seed=0, dev_graph=None, device_weights=None, strict_counts=True, **pp):
    """Returns (device report, oracle result, mask report). The mask report
    is an int (final-mask mismatches after lock-step adoption, asserted 0)
    with .adopted = near-threshold edges the device decided differently."""
    sch = SCHEMES[scheme]
    cfg = ggb.EngineConfig(scheme, sigma, theta, alpha, max_iterations, seed)
    graph = dev_graph if dev_graph is not None else to_graph(ggb, g, device_weights)
    program = device_program(ggb, prog, **pp)
    plain = Oracle.run(g, prog, scheme=sch, sigma=sigma, theta=theta, alpha=alpha,
                       max_iterations=max_iterations, seed=seed, **pp)
    if plain.status == 2:
        try:
            ggb.run(graph, program, cfg)
        except ggb.EngineError as e:
            assert (e.iteration, e.vertex) == (plain.err_iteration, plain.err_vertex), (
                (e.iteration, e.vertex), (plain.err_iteration, plain.err_vertex))
            return None, plain, MaskReport(0)
        raise AssertionError(f"device run did not raise EngineError ({plain.msg})")
    assert plain.status == 0, plain.msg
    rep = ggb.run(graph, program, cfg, want_flags=True)
    ref, mr = lockstep(ggb, g, prog, graph, program, cfg, rep, **pp)
    assert mr.real == 0, f"{mr.real} flags differ outside the near-threshold band: {mr.per_superstep}"
    assert int(mr) == 0, f"{int(mr)} final flags differ after lock-step ({mr.per_superstep})"
    if mr.adopted:
        print(f"near-threshold edges decided differently by the device: {mr.adopted} "
              f"({mr.near} edges in the band)")
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
    if not mr.adopted:  # no adoption: the lock-step run IS the plain oracle run
        assert ref.processed_edges == plain.processed_edges
    return rep, ref, mr
