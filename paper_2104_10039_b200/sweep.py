"""Sweep protocol of the reference (bench.hpp / bench.cpp) on the device engine.

The comparison protocol is what makes "accuracy equal to the reference's"
checkable:
  * the accurate reference runs once per seed (bench.cpp:131-153);
  * every (scheme, sigma, theta, alpha) cell runs with max_iterations = that
    seed's accurate iterations_run (bench.cpp:173);
  * accuracy = (1 - metric error) * 100 with the algorithm's default metric
    (topk for pr/bp with k = max(1, N/100), relative for wcc, stretch for
    sssp; bench.cpp:125-126, :249-257), averaged over seeds;
  * edge_ratio = cell processed edges / accurate processed edges;
  * CSV with the fixed 13-column header (bench.cpp:298-310).

`run_sweep` takes a `runner(graph, program, EngineConfig) -> RunReport`
(default: the device engine), so the same protocol also drives the CPU
oracle in the tests. `plan.graph` may be a host `Graph` (uploaded once) or
a resident `DeviceGraph` (e.g. a device R-MAT at a BASELINE scale; WCC's
symmetrized input is then built on the device too), so a sweep at scale
never moves the graph or any property vector through the host.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import engine as E

ALGOS = ("pr", "sssp", "wcc", "bp")
SCHEME_ORDER = {"accurate": 0, "sp": 1, "sms": 2, "gg": 3}


def default_metric(algo: str) -> str:  # bench.cpp:249-257
    return {"pr": "topk", "bp": "topk", "wcc": "relative", "sssp": "stretch"}[algo]


def default_iteration_budget(algo: str, n: int) -> int:  # bench.cpp:259-267
    return {"pr": 50, "bp": 30}.get(algo, n + 1)


@dataclass
class SweepPlan:  # bench.hpp:32-56
    algo: str = "pr"
    graph: E.Graph | None = None
    graph_label: str = "graph"
    schemes: list = field(default_factory=list)
    sigma_grid: list = field(default_factory=lambda: [0.5])
    theta_grid: list = field(default_factory=lambda: [0.0])
    alpha_grid: list = field(default_factory=lambda: [1])
    iterations: int = 0
    repeats: int = 5
    seeds: list = field(default_factory=lambda: [1])
    threads: int = 1
    topk: int = 0
    metric_override: str | None = None
    sssp_source: int = 0
    sssp_graded: bool = False
    pr_damping: float = 0.85
    epsilon: float = -1.0
    bp_states: int = 2
    bp_coupling: float = 0.8


@dataclass
class SweepRow:  # bench.hpp:58-70
    scheme: str = "accurate"
    sigma: float = 1.0
    theta: float = 0.0
    alpha: int = 0
    iters: int = 0
    repeats: int = 1
    accuracy: float = 100.0
    speedup: float = 1.0
    edge_ratio: float = 1.0
    wall_ms_mean: float = 0.0
    wall_ms_ref: float = 0.0


def _program_and_projection(plan: SweepPlan):  # bench.cpp:269-296
    if plan.algo == "pr":
        eps = 1e-7 if plan.epsilon < 0 else plan.epsilon
        return E.pagerank_spec(plan.pr_damping, eps), plan.graph, lambda p: np.asarray(p, np.float64)
    if plan.algo == "sssp":
        return (E.sssp_spec(plan.sssp_source, plan.sssp_graded), plan.graph,
                lambda p: np.asarray(p, np.float64))
    if plan.algo == "wcc":
        g = plan.graph.symmetrized() if isinstance(plan.graph, E.DeviceGraph) else symmetrized(plan.graph)
        return E.wcc_spec(), g, lambda p: np.asarray(p, np.float64)
    if plan.algo == "bp":
        eps = 1e-6 if plan.epsilon < 0 else plan.epsilon
        return (E.bp_spec(plan.bp_states, plan.bp_coupling, eps), plan.graph,
                lambda p: np.asarray(p, np.float64)[:, 0])
    raise ValueError(f"unknown algorithm: {plan.algo}")


def symmetrized(g: E.Graph) -> E.Graph:
    """graph.cpp:249-257: per destination, its in-edges (in order) followed by
    its out-edges in ascending original-destination order (stable)."""
    n, e = g.n, g.num_edges()
    deg = np.diff(g.in_offsets.astype(np.int64))
    dst = np.repeat(np.arange(n, dtype=np.int64), deg)
    src = g.in_sources.astype(np.int64)
    all_src = np.concatenate([src, dst])
    all_dst = np.concatenate([dst, src])
    order = np.argsort(all_dst, kind="stable")
    w = None
    if g.weights is not None:
        w = np.concatenate([g.weights, g.weights])[order]
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(np.bincount(all_dst, minlength=n), out=off[1:])
    return E.Graph(n, off, all_src[order].astype(np.uint32), w)


def _score(metric, k, approx, exact):  # bench.cpp:68-77
    if metric == "topk":
        return E.topk_error(approx, exact, k)
    if metric == "relative":
        return E.relative_error(approx, exact)
    return E.stretch_error(approx, exact)


def _expand_cells(plan: SweepPlan):  # bench.cpp:33-59
    cells = []
    for s in sorted(set(plan.schemes), key=lambda x: SCHEME_ORDER[x]):
        if s == "accurate":
            continue
        for sigma in plan.sigma_grid:
            if s == "sp":
                cells.append((s, sigma, 0.0, 0))
                continue
            for theta in plan.theta_grid:
                for alpha in plan.alpha_grid:
                    cells.append((s, sigma, theta, alpha))
    cells.sort(key=lambda c: (SCHEME_ORDER[c[0]], c[1], c[2], c[3]))
    return cells


def run_sweep(plan: SweepPlan, runner=None) -> list:
    """bench.cpp:113-227 (sequential cells)."""
    if not plan.seeds:
        raise ValueError("sweep needs >= 1 seed")
    if plan.repeats < 1:
        raise ValueError("repeats must be >= 1")
    if not (plan.sigma_grid and plan.theta_grid and plan.alpha_grid):
        raise ValueError("sweep grids must be non-empty")
    program, graph, project = _program_and_projection(plan)
    n = graph.n
    dev = owned = None
    if runner is None:  # device engine: the graph stays resident for all cells;
        # properties stay in HBM and the metric runs on the GPU (metrics.cu)
        if isinstance(graph, E.DeviceGraph):
            dev = graph
            owned = graph if graph is not plan.graph else None  # a device-built symmetrization
        else:
            dev = owned = E.DeviceGraph.upload(graph)
        runner = lambda _g, p, c: E.run(dev, p, c, device_output=True)  # noqa: E731
        project = lambda _p: dev.last_projection()  # noqa: E731
    elif isinstance(graph, E.DeviceGraph):
        raise TypeError("a custom runner needs a host Graph")
    metric = plan.metric_override or default_metric(plan.algo)
    k = plan.topk if plan.topk > 0 else max(1, n // 100)
    budget = plan.iterations if plan.iterations > 0 else default_iteration_budget(plan.algo, n)
    refs = []
    for seed in plan.seeds:
        cfg = E.EngineConfig("accurate", 1.0, 0.0, 1, budget, seed, plan.threads)
        wall = 0.0
        for _ in range(plan.repeats):
            rep = runner(graph, program, cfg)
            wall += rep.total_wall_seconds
        exact = project(rep.final_properties)
        if dev is not None:
            exact = E.DeviceBuffer.copy(exact)  # outlives the next run
        refs.append((exact, rep.iterations_run, rep.total_processed_edges,
                     wall / plan.repeats * 1e3))
    ref_iters = refs[0][1]
    ref_wall = sum(r[3] for r in refs) / len(refs)
    rows = [SweepRow("accurate", 1.0, 0.0, 0, ref_iters, plan.repeats, 100.0, 1.0, 1.0, ref_wall,
                     ref_wall)]
    for (scheme, sigma, theta, alpha) in _expand_cells(plan):
        acc_sum = ratio_sum = wall_sum = 0.0
        for si, seed in enumerate(plan.seeds):
            cfg = E.EngineConfig(scheme, sigma, theta, max(1, alpha), refs[si][1], seed,
                                 plan.threads)
            wall = 0.0
            for _ in range(plan.repeats):
                rep = runner(graph, program, cfg)
                wall += rep.total_wall_seconds
            acc_sum += _score(metric, k, project(rep.final_properties), refs[si][0]).accuracy
            ratio_sum += 1.0 if refs[si][2] == 0 else rep.total_processed_edges / refs[si][2]
            wall_sum += wall / plan.repeats * 1e3
        ns = len(plan.seeds)
        row = SweepRow(scheme, sigma, theta, alpha, ref_iters, plan.repeats, acc_sum / ns, 1.0,
                       ratio_sum / ns, wall_sum / ns, ref_wall)
        row.speedup = ref_wall / row.wall_ms_mean if row.wall_ms_mean > 0 else 1.0
        rows.append(row)
    if dev is not None:
        for r in refs:
            r[0].close()
    if owned is not None:
        owned.close()
    return rows


def fmt6(v: float) -> str:  # bench.cpp:20-24 ("%.6g")
    if isinstance(v, float) and math.isnan(v):
        return "nan"
    return "%.6g" % v


def emit_csv(rows, plan: SweepPlan) -> str:  # bench.cpp:298-310
    out = ["scheme,algo,graph,sigma,theta,alpha,iters,repeats,accuracy,speedup,edge_ratio,"
           "wall_ms_mean,wall_ms_ref"]
    for r in rows:
        out.append(",".join([r.scheme, plan.algo, plan.graph_label, fmt6(r.sigma), fmt6(r.theta),
                             str(r.alpha), str(r.iters), str(r.repeats), fmt6(r.accuracy),
                             fmt6(r.speedup), fmt6(r.edge_ratio), fmt6(r.wall_ms_mean),
                             fmt6(r.wall_ms_ref)]))
    return "\n".join(out) + "\n"


def mask_time_columns(csv: str) -> str:  # test_bench.cpp:38-64
    lines = csv.splitlines()
    out = [lines[0]]
    for line in lines[1:]:
        cols = line.split(",")
        if len(cols) == 13:
            cols[9] = cols[11] = cols[12] = "X"
        out.append(",".join(cols))
    return "\n".join(out) + "\n"
