"""The partitioned (multi-rank) engine on real device code, one GPU.

Ranks run as host threads of this process, each with its own DeviceGraph
slice and stream, joined by the in-process transport
(gg_exchange_local_group): the same engine code path the NCCL transport
drives across GPUs (partition plan, offset rebase, global-position padding of
each rank's lists, per-iteration slice exchange and counter reduction, the
sparsified list's global base) with host barriers and device copies standing
in for the collectives. No kernel waits on another rank's kernel.

Both exchange paths run: the fused one (default: each vertex kernel stores
its new messages into every rank's replica, here peer buffers on the same
device, with a barrier between the gathers and the vertex kernels) and the
all-gather after the vertex kernel (gg_exchange_set_fused(x, 0)).

The bar is the analogue of test_engine.cpp:161-182: properties and
per-iteration records bit-identical to the single-rank run, for every
program and scheme.
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def _graph(ggb, scale, ef, seed, sym=False, weights=None):
    g = Oracle.rmat(scale, ef, seed)
    if sym:
        g = Oracle.symmetrized(g)
    w = None
    if weights == "u32":
        w = Oracle.rmat_weights_u32(g.e, seed)
    elif weights == "coupling":
        w = Oracle.bp_couplings(g.e, seed)
    return ggb.Graph(g.n, g.off, g.src, w, g.outdeg)


def _program(ggb, prog, graph, seed):
    if prog == "pr":
        return ggb.pagerank_spec(0.85, 1e-7)
    if prog == "sssp":
        return ggb.sssp_spec(int(np.argmax(graph.out_degree)), True)
    if prog == "wcc":
        return ggb.wcc_spec()
    return ggb.EdgeBeliefPropagationProgram(ggb.bp_priors(graph.n, seed), 1e-6)


def _run_ranks(ggb, graph, program, cfg, nranks, fused=True):
    xs = ggb.Exchange.local_group(nranks)
    for x in xs:
        x.set_fused(fused)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            dg = ggb.DeviceGraph.upload(graph, device=0, rank=r, nranks=nranks,
                                        exchange=xs[r].handle)
            out[r] = ggb.run(dg, program, cfg)
            dg.close()
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for x in xs:
        x.close()
    assert not errs, errs
    assert all(r.exchange_fused == (fused and nranks > 1) for r in out)
    return out


def _same(a, b):
    assert a.iterations_run == b.iterations_run
    assert [int(r.mode) for r in a.per_iteration] == [int(r.mode) for r in b.per_iteration]
    assert [r.processed_edges for r in a.per_iteration] == [r.processed_edges for r in b.per_iteration]
    assert [r.active_vertices for r in a.per_iteration] == [r.active_vertices for r in b.per_iteration]
    pa, pb = np.asarray(a.final_properties), np.asarray(b.final_properties)
    assert pa.shape == pb.shape
    assert np.array_equal(pa.view(np.uint8), pb.view(np.uint8)), "not bit-identical"


CASES = [  # prog, scale, edge factor, seed, symmetrise, weights, theta
    ("pr", 15, 16, 3, False, None, 0.01),
    ("sssp", 15, 16, 4, False, "u32", 0.05),
    ("wcc", 14, 16, 5, True, None, 0.0),
    ("bp", 14, 16, 6, False, "coupling", 0.01),
    ("pr", 14, 16, 8, False, "u32", 0.01),  # a program that ignores the graph's weights
]


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "allgather"])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=[c[0] + ("-" + c[5] if c[5] else "") for c in CASES])
def test_ranks_bit_identical_to_one_gpu(ggb, case, nranks, fused):
    prog, scale, ef, seed, sym, weights, theta = case
    graph = _graph(ggb, scale, ef, seed, sym, weights)
    program = _program(ggb, prog, graph, seed)
    cfg = ggb.EngineConfig("gg", 0.5, theta, 2, 30, seed)
    single = ggb.run(graph, program, cfg)
    for rep in _run_ranks(ggb, graph, program, cfg, nranks, fused):
        _same(rep, single)


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "allgather"])
@pytest.mark.parametrize("scheme", ["accurate", "sp", "sms", "gg"])
def test_ranks_all_schemes_pagerank(ggb, scheme, fused):
    graph = _graph(ggb, 16, 16, 7)
    program = ggb.pagerank_spec(0.85, 1e-7)
    cfg = ggb.EngineConfig(scheme, 0.5, 0.01, 3, 25, 7)
    single = ggb.run(graph, program, cfg)
    for rep in _run_ranks(ggb, graph, program, cfg, 4, fused):
        _same(rep, single)


def test_ranks_fused_runs_back_to_back(ggb):
    """Several runs (different programs, hence message buffers of different
    sizes) on the same rank graphs: the peer replicas are re-registered when
    the buffer changes and reused otherwise."""
    graph = _graph(ggb, 14, 16, 9)
    progs = [ggb.pagerank_spec(0.85, 1e-7), ggb.wcc_spec(), ggb.pagerank_spec(0.85, 1e-7),
             ggb.sssp_spec(int(np.argmax(graph.out_degree)), True)]
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 2, 12, 9)
    singles = [ggb.run(graph, p, cfg) for p in progs]
    nranks = 3
    xs = ggb.Exchange.local_group(nranks)
    out, errs = [[None] * len(progs) for _ in range(nranks)], []

    def work(r):
        try:
            dg = ggb.DeviceGraph.upload(graph, device=0, rank=r, nranks=nranks, exchange=xs[r].handle)
            for i, p in enumerate(progs):
                out[r][i] = ggb.run(dg, p, cfg)
            dg.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for x in xs:
        x.close()
    assert not errs, errs
    for r in range(nranks):
        for i in range(len(progs)):
            assert out[r][i].exchange_fused
            _same(out[r][i], singles[i])


@pytest.mark.parametrize("nranks", [3, 5])
def test_ranks_with_tiny_and_empty_slices(ggb, nranks):
    """Ranks whose 32-aligned slice is empty or holds no edges (a 70-vertex
    graph over 5 ranks) still take part in every exchange."""
    g = Oracle.power_law(70, 3.0, 2.0, 11)
    graph = ggb.Graph(g.n, g.off, g.src, None, g.outdeg)
    plan = ggb.partition_plan(graph, nranks)
    assert any(plan[r + 1] == plan[r] for r in range(nranks)), plan  # some rank is empty
    for prog in (ggb.pagerank_spec(0.85, 1e-7), ggb.wcc_spec()):
        cfg = ggb.EngineConfig("gg", 0.5, 0.01, 2, 20, 3)
        single = ggb.run(graph, prog, cfg)
        for rep in _run_ranks(ggb, graph, prog, cfg, nranks):
            _same(rep, single)


def test_ranks_agree_on_the_exchange_path(ggb):
    """Ranks asking for different exchange paths (rank 0 fused, the others
    not) agree on the all-gather through the registration's agreement round:
    no rank stores into replicas another rank does not expect."""
    graph = _graph(ggb, 14, 16, 10)
    program = ggb.pagerank_spec(0.85, 1e-7)
    cfg = ggb.EngineConfig("gg", 0.5, 0.01, 2, 12, 10)
    single = ggb.run(graph, program, cfg)
    nranks = 3
    xs = ggb.Exchange.local_group(nranks)
    for r, x in enumerate(xs):
        x.set_fused(r == 0)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            dg = ggb.DeviceGraph.upload(graph, device=0, rank=r, nranks=nranks, exchange=xs[r].handle)
            out[r] = ggb.run(dg, program, cfg)
            dg.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for x in xs:
        x.close()
    assert not errs, errs
    for rep in out:
        assert not rep.exchange_fused
        _same(rep, single)


def test_nccl_transport_selftest_one_rank_communicator(ggb):
    """The NCCL transport's own calls on this GPU: ncclGetUniqueId,
    ncclCommInitRank, the grouped ncclBroadcast all-gather, the sum and max
    all-reduces and ncclCommDestroy run over a one-rank communicator and are
    compared with their closed forms (gg_exchange_selftest). bench.py runs
    the same check on every rank before a multi-GPU measurement."""
    x = ggb.Exchange(0, 1, ggb.Exchange.unique_id())
    try:
        x.selftest()
        x.selftest()  # a second round on the same communicator
    finally:
        x.close()


def test_local_transport_selftest_is_a_noop(ggb):
    xs = ggb.Exchange.local_group(2)
    for x in xs:
        x.selftest()
        x.close()
