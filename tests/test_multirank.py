"""Multi-rank protocol of the destination-partitioned engine, on CPU (gloo).

The device engine (engine.cuh) runs one process per GPU: the product's
partition plan (gg_partition_plan: 32-aligned, edge-balanced destination
ranges), a rank-local iteration over the owned destinations reading the
replicated previous-iteration vector, an AllGatherV of the owned slices and
an allreduce of {gathered, processed, changed, smallest invalid vertex} so
every rank takes the same early-exit / EngineError decision
(engine.hpp:226-240). Here the same protocol runs on 2 gloo ranks with the
CPU oracle's range step as the per-rank compute, and must reproduce the
single-process reference result bit for bit (the analogue of the
reference's thread-count invariance, test_engine.cpp:161-182).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import BP, GG, PR, SMS, SSSP, WCC, Oracle

CASES = [
    ("powerlaw", PR, dict(scheme=GG, sigma=0.5, theta=0.05, alpha=3, max_iterations=40, seed=5), {}),
    ("powerlaw", PR, dict(scheme=SMS, sigma=0.4, theta=0.1, alpha=2, max_iterations=40, seed=2), {}),
    ("weighted", SSSP, dict(scheme=GG, sigma=0.5, theta=0.05, alpha=2, max_iterations=200, seed=3),
     dict(graded=True)),
    ("sym", WCC, dict(scheme=GG, sigma=0.5, theta=0.0, alpha=2, max_iterations=200, seed=4), {}),
    ("powerlaw", BP, dict(scheme=GG, sigma=0.6, theta=0.01, alpha=3, max_iterations=30, seed=6), {}),
]


def make_graph(kind):
    if kind == "powerlaw":
        return Oracle.power_law(1200, 7.0, 2.1, 9)
    if kind == "weighted":
        return Oracle.random_graph(900, 7000, 4, True)
    return Oracle.symmetrized(Oracle.power_law(800, 5.0, 2.2, 3))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_main(rank, world, port, case_idx, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2104_10039_b200 as ggb
    kind, prog, cfg, pp = CASES[case_idx]
    g = make_graph(kind)
    bounds = ggb.partition_plan(ggb.Graph(g.n, g.off, g.src), world).astype(np.int64)
    vb, ve = int(bounds[rank]), int(bounds[rank + 1])
    st = Oracle.Stepper(g, prog, **pp)
    prev = st.init_props()
    nxt = np.empty_like(prev)
    flags = (np.ones(g.e, np.uint8) if cfg["scheme"] == 0
             else Oracle.sparsify(g.e, cfg["sigma"], cfg["seed"]))
    aid = np.array([flags[g.off[v]:g.off[v + 1]].sum() for v in range(g.n)], np.uint32)
    status = np.ones(g.n, np.uint8)
    status_next = np.zeros(g.n, np.uint8)
    recs, err = [], None
    row_bytes = prev.reshape(g.n, -1)[0].nbytes
    width = int(np.diff(bounds).max())
    for t in range(1, cfg["max_iterations"] + 1):
        mode = int(ggb.mode_for(cfg["scheme"], t, cfg["alpha"]))
        ctr = st.step(mode, cfg["theta"], flags, aid, prev, status, nxt, status_next, vb, ve)
        # AllGatherV of the owned slices (padded all_gather) of next and status
        mine = np.zeros((width, row_bytes), np.uint8)
        mine[:ve - vb] = nxt.reshape(g.n, -1)[vb:ve].view(np.uint8).reshape(ve - vb, row_bytes)
        parts = [torch.zeros((width, row_bytes), dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        flat = nxt.reshape(g.n, -1).view(np.uint8).reshape(g.n, row_bytes)
        for r in range(world):
            flat[bounds[r]:bounds[r + 1]] = parts[r][:bounds[r + 1] - bounds[r]].numpy()
        # counters: sum gathered/processed, max changed, min (1-based) bad vertex
        c = torch.tensor([int(ctr[0]), int(ctr[1]), int(ctr[2])], dtype=torch.int64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        bad = torch.tensor([int(ctr[3]) if ctr[3] else 1 << 62], dtype=torch.int64)
        dist.all_reduce(bad, op=dist.ReduceOp.MIN)
        if bad.item() < (1 << 62):
            err = (t, int(bad.item()) - 1)
            break
        recs.append((mode, int(c[0]), int(c[1])))
        prev, nxt = nxt, prev
        status, status_next = status_next, status
        # only the owned status slice matters to this rank (skip test is local)
        if int(c[2]) == 0:
            break
    st.close()
    if rank == 0:
        out.put((prev.tobytes(), recs, err))
    dist.destroy_process_group()


@pytest.mark.parametrize("case_idx", range(len(CASES)))
def test_two_rank_protocol_bit_identical(case_idx):
    kind, prog, cfg, pp = CASES[case_idx]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=rank_main, args=(r, 2, port, case_idx, q)) for r in range(2)]
    for p in procs:
        p.start()
    props, recs, err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = Oracle.run(make_graph(kind), prog, **cfg, **pp)
    assert err is None and ref.status == 0
    assert props == ref.props.tobytes()
    assert [r[0] for r in recs] == ref.modes
    assert [r[1] for r in recs] == ref.processed_edges
    assert [r[2] for r in recs] == ref.active_vertices
