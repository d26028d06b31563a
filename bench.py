#!/usr/bin/env python
"""bench.py — GTEPS of the GraphGuess approximate pull-gather engine on B200.

A STEP is one complete engine run (gg::run, engine.hpp:141-249) of the
workload's program on its synthetic R-MAT graph: gg scheme (sigma 0.5,
alpha 4, the workload's theta), max_iterations = the accurate run's
iterations_run (bench.cpp:173 protocol). value = processed edges of all
ranks / max-over-ranks device time, in GTEPS.

Workloads (BASELINE.json configs; data are seeded synthetic R-MAT graphs
built on the device — the paper's datasets are not used):
  c1 PR   s16 EF16 seed 1             c2 SSSP s22 EF16 seed 2, u32 w, graded
  c3 WCC  s23 EF16 seed 3, symmetrised c4 BP  s25 EF16 seed 4, fp32 c_e/priors
  c5 PR   s26 EF28 seed 5 (default: the largest graph; multi-GPU scaling)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
      N > 1 without torchrun: re-launches itself under torch.distributed.run
      (one process per GPU, NCCL transport); under torchrun WORLD_SIZE must
      equal N.
  python bench.py --gpus N --transport local
      N ranks as host threads sharing ONE GPU (in-process transport): runs
      the partitioned engine end to end (exchange bytes and time per
      iteration are reported); not a scaling measurement (n_gpus = 1).
  python bench.py --impl reference ...   (reference CPU engine, rank 0 only)

Beside the device number the line carries: accuracy of the gg run against
the accurate run (the reference sweep's score, bench.cpp:181-190) and its
edge ratio; the roofline of the dominant kernel; the end-to-end figure
through the public API with host buffers; the reference CPU engine on a
bounded sample (cpu_baseline, rank 0 at N = 1).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

# Both CPU legs (cpu_baseline and --impl reference) run the reference's
# OpenMP loops under the same settings; set before any OpenMP runtime loads.
os.environ.setdefault("OMP_WAIT_POLICY", "passive")
os.environ.setdefault("OMP_PROC_BIND", "close")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS of full and sparsified gather iterations; % of HBM roofline"
GATHER_PEAK_G = 264.3  # G random 8-byte gathers/s, one B200 (profiles/r2_dsmem_gather_bench.txt)
WORKLOADS = {
    "c1": dict(prog="pr", scale=16, ef=16, seed=1, theta=0.01, weights=None, sym=False),
    "c2": dict(prog="sssp", scale=22, ef=16, seed=2, theta=0.05, weights="u32", sym=False),
    "c3": dict(prog="wcc", scale=23, ef=16, seed=3, theta=0.0, weights=None, sym=True),
    "c4": dict(prog="bp", scale=25, ef=16, seed=4, theta=0.01, weights="coupling", sym=False),
    "c5": dict(prog="pr", scale=26, ef=28, seed=5, theta=0.01, weights=None, sym=False),
}
SIGMA, ALPHA = 0.5, 4
DTYPE = {"pr": "f64", "sssp": "u32", "wcc": "u32", "bp": "f32 storage / f64 arithmetic"}
# bench.cpp:280-287 default metric per algorithm: 0 top-k, 1 relative, 2 stretch
METRIC_KIND = {"pr": 0, "bp": 0, "wcc": 1, "sssp": 2}
METRIC_NAME = {0: "topk", 1: "relative", 2: "stretch"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def omp_env():
    return {k: os.environ.get(k) for k in ("OMP_WAIT_POLICY", "OMP_PROC_BIND")}


def config_json(args, wl, world, transport="nccl"):
    par = f"dst-partition x{world}" + (f" ({transport})" if world > 1 else "")
    return {
        "workload": f"{args.workload}: {wl['prog'].upper()} on R-MAT s{wl['scale']} EF{wl['ef']} "
                    f"seed {wl['seed']}" + (" symmetrised" if wl["sym"] else ""),
        "scale": wl["scale"], "edge_factor": wl["ef"], "seed": wl["seed"],
        "scheme": "gg", "sigma": SIGMA, "theta": wl["theta"], "alpha": ALPHA,
        "rmat_abcd": [0.57, 0.19, 0.19, 0.05], "parallelism": par,
        "l2": "inputs larger than L2 (CSC >> 126 MB)" if wl["scale"] >= 22
              else "L2-resident graph (no flush: launch-bound parity config)",
    }


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    """`nvidia-smi -lms 50` beside the run. It is started BEFORE the warm-up (its
    start-up, tens of ms of driver queries, used to land inside the first timed
    step and stretch a host sync there by several ms); only the samples whose
    timestamps fall inside the timed region [begin(), end()] are reported."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu,timestamp")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def _in_window(self, stamp):
        if self.t0 is None or self.t1 is None:
            return True
        try:
            import datetime
            t = datetime.datetime.strptime(stamp, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except Exception:
            return True
        return self.t0 - 0.05 <= t <= self.t1 + 0.05

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        every = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                every.append(parts)
        os.unlink(self.path)
        rows = [r for r in every if len(r) < 8 or self._in_window(r[7])]
        if not rows and every:  # region shorter than the sampling period: the nearest sample
            rows = every[-1:]
        if not rows:  # region shorter than the sampling period: one immediate sample
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                rows = [[p.strip() for p in line.split(",")] for line in out.splitlines()
                        if len(line.split(",")) >= 7]
            except Exception:
                rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r[6].isdigit() and int(r[6]) > 0] or rows
        sm = [int(r[0]) for r in loaded if r[0].isdigit()]
        mx = [int(r[1]) for r in rows if r[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded)}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def make_program(ggb, wl, dg, n, host_priors=None):
    """The workload's program. C4's fp32 prior table is a program input like
    the graph: resident in HBM for the device-timed runs (generated there),
    a host array (host_priors) on the end-to-end path."""
    if wl["prog"] == "pr":
        return ggb.pagerank_spec(0.85, 1e-7)
    if wl["prog"] == "sssp":
        od = dg.out_degree()
        return ggb.sssp_spec(int(od.argmax()), True)  # highest out-degree vertex
    if wl["prog"] == "wcc":
        return ggb.wcc_spec()
    pri = host_priors if host_priors is not None else ggb.bp_priors(n, wl["seed"], device=True)
    return ggb.EdgeBeliefPropagationProgram(pri, 1e-6)


def budget_for(wl, n):
    # bench.cpp:259-267 default budgets: pr 50, bp 30, sssp/wcc N+1
    return {"pr": 50, "bp": 30}.get(wl["prog"], n + 1)


def prop_bytes(wl):
    return {"pr": 8, "sssp": 8, "wcc": 4, "bp": 16}[wl["prog"]]


def msg_bytes(wl):  # per-vertex message the exchange carries
    return {"pr": 8, "sssp": 4, "wcc": 4, "bp": 8}[wl["prog"]]


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def load_traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/ncu_<workload>.json), if one exists."""
    p = os.path.join(ROOT, "profiles", f"ncu_{workload}.json")
    try:
        d = json.load(open(p))
        return d.get("dominant_kernel_dram_bytes_per_launch"), d
    except Exception:
        return None, None


def load_mask_parity(workload):
    """Active-edge mask parity of this workload at full size against the lock-step
    oracle: the record written by tests/test_gpu_full_size.py (GGB_PARITY_OUT) on
    a B200 and committed as profiles/mask_parity.json. North-star: masks identical
    except edges whose influence lies within rounding of theta, their count reported."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "mask_parity.json")))[workload]
    except Exception:
        return None
    return d | {"source": "profiles/mask_parity.json (tests/test_gpu_full_size.py, lock-step oracle, "
                          "every flag after every superstep)"}


def device_accuracy(ggb, wl, n, acc_proj, dg, rep, acc_edges):
    """Score of the gg run against the accurate run on the device (the
    reference sweep's metric per algorithm, bench.cpp:181-190 / :280-287);
    both projections stay in HBM."""
    kind = METRIC_KIND[wl["prog"]]
    proj = dg.last_projection()
    if kind == 0:
        r = ggb.topk_error(proj, acc_proj, max(1, n // 100))
    elif kind == 1:
        r = ggb.relative_error(proj, acc_proj)
    else:
        r = ggb.stretch_error(proj, acc_proj)
    return {"metric": METRIC_NAME[kind], "accuracy": round(r.accuracy, 6),
            "k": max(1, n // 100) if kind == 0 else None,
            "edge_ratio": round(rep.total_processed_edges / acc_edges, 6) if acc_edges else 1.0}


def summarize(args, wl, reps, info, e, per_rank_frac, peak_info):
    per = [it for r in reps for it in r.per_iteration]
    approx = [it for it in per if it.mode.name == "approximate"]
    full = [it for it in per if it.mode.name != "approximate"]

    def gteps(its):  # gather step (edge + vertex kernels) of this rank
        t = sum(i.kernel_ms for i in its)
        return (sum(i.processed_edges for i in its) * per_rank_frac / (t / 1e3) / 1e9) if t else None

    def gbs(its, b="edge_bytes", m="edge_ms"):  # algorithmic bytes / CUDA-event time
        t = sum(getattr(i, m) for i in its)
        return (sum(getattr(i, b) for i in its) / (t / 1e3) / 1e9) if t else None

    peak, peak_src = peak_info
    dom = approx if approx else full  # the dominant kernel: the approximate edge gather
    achieved = gbs(dom)
    traffic, ncu = load_traffic(args.workload)
    roofline = {
        "bound": "hbm", "kernel": "edge_kernel<kEdgePlain> (approximate gather, sparsified CSC)"
        if approx else "edge_kernel (full gather)",
        "achieved": round(achieved, 1) if achieved else None, "peak": peak, "peak_source": peak_src,
        "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": traffic,
        "traffic_source": (f"profiles/ncu_{args.workload}.json: ncu --set full, dram read+write of one "
                           f"launch with {ncu['dominant_kernel_algo_bytes_per_launch']} algorithmic bytes"
                           if ncu else None),
        "algo_bytes_per_launch": int(sum(i.edge_bytes for i in dom) / max(len(dom), 1)),
        "bytes_model": "E_p * (4 src + sizeof(message) + sizeof(weight)); SURVEY §8(d) b_e",
        "kernel_ms_per_launch": round(sum(i.edge_ms for i in dom) / max(len(dom), 1), 4),
        "launches": len(dom),
        "vertex_kernel_gbs": round(gbs(per, "vertex_bytes", "vertex_ms"), 1)
        if gbs(per, "vertex_bytes", "vertex_ms") else None,
        "full_gather_edge_gbs": round(gbs(full), 1) if gbs(full) else None,
    }
    # The gather's second ceiling: every random message gather is one L1TEX
    # tag lookup, ~0.9 per clock per SM on B200 whatever cache level serves it
    # (tools/dsmem_gather_bench.cu, `ldg` rows of profiles/r2_dsmem_gather_bench.txt;
    # shared-memory, DSMEM and TMA gather4 paths do not add to it, r2_summary.md).
    t_dom = sum(i.edge_ms for i in dom)
    # (PageRank only: 8-byte messages gathered with plain loads; the 4-byte
    # programs also serve hot slots from shared memory, BP's gather is ALU-heavy)
    if t_dom and wl["prog"] == "pr":
        ach = sum(i.processed_edges for i in dom) * per_rank_frac / (t_dom / 1e3) / 1e9
        roofline["gather_request_bound"] = {
            "unit": "G gathers/s", "achieved": round(ach, 1), "peak": GATHER_PEAK_G,
            "frac": round(ach / GATHER_PEAK_G, 4),
            "peak_source": "measured pure LDG gather rate on the hot-first R-MAT s26 slot stream "
                           "(profiles/r2_dsmem_gather_bench.txt, 256-thread CTAs)",
            "hbm_frac_at_peak": round(GATHER_PEAK_G * (sum(i.edge_bytes for i in dom) /
                                      max(sum(i.processed_edges for i in dom) * per_rank_frac, 1)) / peak, 4)
            if peak else None}
    return roofline, gteps(approx), gteps(full), per


def exchange_stats(ggb, wl, world, per, host_out_degree, bounds, fused=False):
    """NVLink bytes each rank receives per iteration (the gathered message
    slots of the other ranks' ranges) and the measured
    exchange time per iteration (CUDA events around it, this rank)."""
    import numpy as np
    if world <= 1:
        return None
    od = host_out_degree
    gathered = [int(np.count_nonzero(od[int(bounds[r]):int(bounds[r + 1])])) for r in range(world)]
    total = sum(gathered)
    recv = [(total - gathered[r]) * msg_bytes(wl) for r in range(world)]
    ex = [it.exchange_ms for it in per if it.exchange_ms]
    return {"bytes_received_per_iter_per_rank": recv, "max_bytes_received_per_iter": max(recv),
            "exchange_ms_per_iter_rank0": round(sum(ex) / len(ex), 4) if ex else None,
            "what": "message slots with out-degree > 0 of the other ranks' ranges",
            "path": ("fused: the vertex kernel stores them into every rank's replica (peer "
                     "memory), one barrier between gathers and vertex kernels; exchange_ms = "
                     "the counter all-reduce" if fused else
                     "all-gather after the vertex kernel (grouped ncclBroadcast = AllGatherV)")}


def ours(args):
    import numpy as np
    import torch

    import paper_2104_10039_b200 as ggb

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    torch.cuda.set_device(local)
    dist = None
    exchange = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [ggb.Exchange.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        exchange = ggb.Exchange(rank, world, uid[0])
        exchange.set_fused(not args.no_fused)
        exchange.selftest()  # ragged all-gather + all-reduces against closed forms, before any work
    wl = WORKLOADS[args.workload]
    t_setup = time.perf_counter()
    dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"],
                              weights=wl["weights"], device=local, rank=rank, nranks=world,
                              exchange=exchange.handle if exchange else None)
    n, e = dg.n, dg.e
    info = dg.info()
    program = make_program(ggb, wl, dg, n)
    clocks = ClockSampler(local)
    clocks.start()  # before the accurate run and the warm-up: see ClockSampler
    acc = ggb.run(dg, program, ggb.EngineConfig("accurate", max_iterations=budget_for(wl, n)),
                  device_output=True)
    acc_proj = ggb.DeviceBuffer.copy(dg.last_projection())
    budget = acc.iterations_run
    cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, budget, wl["seed"])
    log(f"[rank {rank}] graph n={n} e={e} local={info} accurate iterations={budget} "
        f"setup {time.perf_counter() - t_setup:.1f}s")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        ggb.run(dg, program, cfg, device_output=True)
    barrier()
    clocks.begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    reps = [ggb.run(dg, program, cfg, timing=True, device_output=True) for _ in range(args.steps)]
    ev1.record()
    barrier()
    clocks.end()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    edges = sum(r.total_processed_edges for r in reps)
    value = edges / (ms / 1e3) / 1e9
    launches = sum(r.kernel_launches for r in reps)

    # accuracy of the (last) gg run against the accurate run, on the device
    accuracy = device_accuracy(ggb, wl, n, acc_proj, dg, reps[-1], acc.total_processed_edges)
    acc_proj.close()

    peaks = load_peaks()
    peak_info = (peaks.get("hbm_gbs", 6650.0),
                 "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)" if "hbm_gbs" in peaks
                 else "fallback 6650 GB/s (B200_PROFILING.md)")
    roofline, g_sp, g_full, per = summarize(args, wl, reps, info, e, info["e_local"] / max(e, 1),
                                            peak_info)

    # ---- end to end through the public API: pinned host CSC -> H2D upload
    # (gg_dev_graph_create), run, D2H of the final properties, every step.
    e2e = None
    host = None
    if not args.no_e2e or world > 1:
        def pinned(count, dt):
            t = torch.empty(int(count) * np.dtype(dt).itemsize, dtype=torch.uint8,
                            pin_memory=True)
            return t.numpy().view(dt)
        if world == 1:
            host = dg.to_host(alloc=pinned)
        else:
            full_g = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"],
                                          weights=wl["weights"], device=local)
            host = full_g.to_host(alloc=pinned)
            full_g.close()
    if not args.no_e2e:
        wsz = host.weights.dtype.itemsize if host.weights is not None else 0
        h2d = (info["v_end"] - info["v_begin"] + 1) * 8 + info["e_local"] * (4 + wsz) + n * 4
        d2h = n * prop_bytes(wl)
        program_e2e = program
        if wl["prog"] == "bp":  # the prior table travels with every step
            pri = pinned(2 * n, np.float32).reshape(n, 2)
            pri[:] = ggb.bp_priors(n, wl["seed"])
            program_e2e = make_program(ggb, wl, dg, n, host_priors=pri)
            h2d += pri.nbytes

        out_shape = {"pr": (n,), "sssp": (n,), "wcc": (n,), "bp": (n, 2)}[wl["prog"]]
        out_dt = np.uint32 if wl["prog"] == "wcc" else np.float64
        out_buf = pinned(int(np.prod(out_shape)), out_dt).reshape(out_shape)

        def e2e_step():
            # the graph is uploaded for this run (gg::run(Graph, ...)): its
            # initial sparsification overlaps the upload on one rank
            g2 = ggb.DeviceGraph.upload(host, device=local, rank=rank, nranks=world,
                                        exchange=exchange.handle if exchange else None,
                                        for_run=cfg if world == 1 else None)
            r = ggb.run(g2, program_e2e, cfg, out=out_buf)
            g2.close()
            return r
        for _ in range(args.warmup):
            e2e_step()
        barrier()
        ev0.record()
        e2e_reps = [e2e_step() for _ in range(args.steps)]
        ev1.record()
        barrier()
        ems = ev0.elapsed_time(ev1)
        if dist:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        ee = sum(r.total_processed_edges for r in e2e_reps)
        e2e = {"value": round(ee / (ems / 1e3) / 1e9, 4), "unit": "GTEPS",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(ems / args.steps, 3),
               "path": "gg_dev_graph_create (pinned host CSC) + gg_run_* + D2H properties"}

    xstats = None
    if world > 1:
        xstats = exchange_stats(ggb, wl, world, per, host.out_degree,
                                ggb.partition_plan(host, world), reps[0].exchange_fused)

    # ---- reference CPU path beside it (rank 0, N=1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if host is None:
            host = dg.to_host()
        cpu = cpu_baseline_sample(wl, host)

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPE[wl["prog"]], "data": "synthetic R-MAT (seeded, built on device)",
        # config is the workload only and identical on both arms; the shape of a
        # step (which differs: a whole gg run here, a bounded sample there) is "step"
        "config": config_json(args, wl, world) | {"vertices": n, "edges": e},
        "step": {"what": "one whole gg run (sparsify, every iteration, early exit)",
                 "max_iterations": budget, "iterations_per_step": reps[0].iterations_run,
                 "edges_per_step": reps[0].total_processed_edges},
        "gteps_sparsified_kernel": round(g_sp, 3) if g_sp else None,
        "gteps_full_kernel": round(g_full, 3) if g_full else None,
        "accuracy": accuracy,
        "mask_parity": load_mask_parity(args.workload),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk,
        # per iteration of one run: processed edges / vertices (engine.hpp:186-189,
        # `active_vertices` = the vertices that passed the skip test) and the
        # edge / vertex kernel times (CUDA events, engine stream)
        "per_iteration": [{"mode": it.mode.name, "edges": it.processed_edges,
                           "vertices": it.active_vertices,
                           "vertex_frac": round(it.active_vertices / n, 4) if n else None,
                           "edge_ms": round(it.edge_ms, 3), "vertex_ms": round(it.vertex_ms, 3),
                           "rebuild_ms": round(it.rebuild_ms, 3)}
                          for it in reps[0].per_iteration],
    }
    if xstats:
        out["exchange"] = xstats
    if rank == 0:
        print(json.dumps(out), flush=True)
    if exchange:
        dg.close()
        exchange.close()
    if dist:
        dist.destroy_process_group()


def ours_local(args):
    """N ranks as host threads on one GPU through the in-process transport
    (gg_exchange_local_group): the whole partitioned engine path, exchange
    included, on one device. Graph slices are created one rank at a time
    (bounded peak memory); the timed runs of all ranks overlap."""
    import torch

    import paper_2104_10039_b200 as ggb

    N = args.gpus
    wl = WORKLOADS[args.workload]
    torch.cuda.set_device(0)
    xs = ggb.Exchange.local_group(N)
    for x in xs:
        x.set_fused(not args.no_fused)
    create_lock = threading.Lock()
    res = [None] * N
    errs = []
    start = threading.Barrier(N)

    def work(r):
        try:
            with create_lock:
                dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"],
                                          weights=wl["weights"], device=0, rank=r, nranks=N,
                                          exchange=xs[r].handle)
            program = make_program(ggb, wl, dg, dg.n)
            acc = ggb.run(dg, program, ggb.EngineConfig("accurate",
                                                       max_iterations=budget_for(wl, dg.n)),
                          device_output=True)
            cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, acc.iterations_run, wl["seed"])
            for _ in range(args.warmup):
                ggb.run(dg, program, cfg, device_output=True)
            start.wait()
            t0 = time.perf_counter()
            reps = [ggb.run(dg, program, cfg, timing=True, device_output=True)
                    for _ in range(args.steps)]
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            res[r] = dict(info=dg.info(), reps=reps, wall=wall, budget=acc.iterations_run,
                          n=dg.n, e=dg.e, od=dg.out_degree() if r == 0 else None)
            dg.close()
        except BaseException as ex:  # noqa: BLE001
            errs.append(ex)
            try:
                start.abort()
            except Exception:
                pass
    ts = [threading.Thread(target=work, args=(r,)) for r in range(N)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for x in xs:
        x.close()
    if errs:
        raise errs[0]
    n, e = res[0]["n"], res[0]["e"]
    wall = max(r["wall"] for r in res)
    edges = sum(rep.total_processed_edges for rep in res[0]["reps"])  # every rank reports the total
    per = [it for rep in res[0]["reps"] for it in rep.per_iteration]
    import numpy as np
    bounds = [0]
    for r in res:
        bounds.append(r["info"]["v_end"])
    xstats = exchange_stats(ggb, wl, N, per, res[0]["od"], np.array(bounds, np.uint64),
                            res[0]["reps"][0].exchange_fused)
    xstats["exchange_ms_per_iter_per_rank"] = [
        round(sum(it.exchange_ms for rep in r["reps"] for it in rep.per_iteration) /
              max(1, sum(len(rep.per_iteration) for rep in r["reps"])), 4) for r in res]
    out = {
        "metric": METRIC, "value": round(edges / wall / 1e9, 4), "unit": "GTEPS", "n_gpus": 1,
        "ranks": N, "transport": "local: ranks are host threads sharing one GPU (host barriers + "
                                 "device copies); not a scaling measurement",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPE[wl["prog"]], "data": "synthetic R-MAT (seeded, built on device)",
        "config": config_json(args, wl, N, "local") | {
            "vertices": n, "edges": e, "max_iterations": res[0]["budget"],
            "iterations_per_step": res[0]["reps"][0].iterations_run,
            "edges_per_rank": [r["info"]["e_local"] for r in res],
            "vertex_ranges": [[r["info"]["v_begin"], r["info"]["v_end"]] for r in res]},
        "exchange": xstats,
        "timing": "host wall clock around the ranks' runs (threads share one device)",
        "gpu_launches": sum(rep.kernel_launches for r in res for rep in r["reps"]),
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------
# reference CPU engine (the unmodified reference, oracle/_ref/libggref.so)
# --------------------------------------------------------------------------
def ref_inputs(wl, host_graph=None):
    """Host CSC for the reference: from our arm's export, else the CPU
    generator (same R-MAT specification, oracle/gg_oracle.c)."""
    import numpy as np

    from oracle.oracle import CSC, Oracle
    if host_graph is not None:
        w = host_graph.weights.astype(np.float64) if host_graph.weights is not None else None
        return CSC(host_graph.n, host_graph.in_offsets, host_graph.in_sources, w,
                   host_graph.out_degree)
    g = Oracle.rmat(wl["scale"], wl["ef"], wl["seed"], threads=os.cpu_count() or 1)
    if wl["sym"]:
        g = Oracle.symmetrized(g)
    if wl["weights"] == "u32":
        g.w = Oracle.rmat_weights_u32(g.e, wl["seed"]).astype(np.float64)
    elif wl["weights"] == "coupling":
        g.w = Oracle.bp_couplings(g.e, wl["seed"]).astype(np.float64)
    return g


def ref_params(wl, g):
    import numpy as np

    from oracle.oracle import BP_EDGE, PR, SSSP, WCC, Oracle
    if wl["prog"] == "pr":
        return PR, dict(damping=0.85, epsilon=1e-7)
    if wl["prog"] == "sssp":
        return SSSP, dict(source=int(np.argmax(g.outdeg)), graded=True)
    if wl["prog"] == "wcc":
        return WCC, {}
    return BP_EDGE, dict(prior_table=Oracle.bp_priors(g.n, wl["seed"]), epsilon=1e-6)


STEP_ITERS = 1            # --impl reference: each step = the first (approximate) iteration
WINDOW_ITERS = ALPHA + 1  # cpu_baseline: one window of alpha approximate iterations + a superstep


def _mode_gteps(r, mode):
    e = sum(pe for m, pe in zip(r.modes, r.processed_edges) if m == mode)
    w = sum(ws for m, ws in zip(r.modes, r.wall_seconds) if m == mode)
    return (round(e / w / 1e9, 5) if w else None), e, w


def reference_window(wl, g, handle=None, threads=None, iters=WINDOW_ITERS):
    """The reference gg::run on the workload capped at `iters` iterations
    (default: alpha approximate iterations + one superstep); per-mode GTEPS
    from its own RunReport (processed_edges / wall_seconds per iteration)."""
    from oracle.oracle import GG, Reference
    prog, pp = ref_params(wl, g)
    cores = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    r = Reference.run(g, prog, scheme=GG, sigma=SIGMA, theta=wl["theta"], alpha=ALPHA,
                      max_iterations=iters, seed=wl["seed"], threads=cores, handle=handle, **pp)
    elapsed = time.perf_counter() - t0
    assert r.status == 0, r.msg
    sp, esp, wsp = _mode_gteps(r, 0)
    full, efu, wfu = _mode_gteps(r, 2)
    wall = sum(r.wall_seconds)
    return {"value": round(r.total_processed_edges / wall / 1e9, 5) if wall else None,
            "sparsified": sp, "full": full, "iterations": r.iterations_run,
            "edges": r.total_processed_edges, "elapsed_s": round(elapsed, 2), "cores": cores}


def reference_one_thread(wl, g, frac=16):
    """1-thread reference rate on a bounded sample: the destination prefix
    holding ~E/frac in-edges (all sources still range over every vertex, so
    the gathers touch the whole property array), first iteration."""
    from oracle.oracle import CSC
    import numpy as np
    k = int(np.searchsorted(g.off, g.off[-1] // frac))
    sub = CSC(g.n, np.concatenate([g.off[:k + 1], np.full(g.n - k, g.off[k], np.uint64)]),
              g.src[:int(g.off[k])], None if g.w is None else g.w[:int(g.off[k])])
    r = reference_window(wl, sub, threads=1, iters=1)
    r["sample"] = (f"destinations [0, {k}) ({int(g.off[k])} in-edges, 1/{frac} of E; sources over all "
                   f"{g.n} vertices), first iteration, 1 thread")
    return r


def cpu_baseline_sample(wl, host_graph):
    """cpu_baseline of our arm: the reference engine on the same graph,
    all host threads, one window of alpha approximate iterations plus one
    superstep (~30 s at c5)."""
    from oracle.oracle import Reference
    if not Reference.available():
        return None
    g = ref_inputs(wl, host_graph)
    w = reference_window(wl, g)
    cores = w["cores"]
    return {"value": w["value"], "unit": "GTEPS", "cores": cores, "kind": "reference",
            "sparsified": w["sparsified"], "full": w["full"],
            "cpu_model": cpu_model(), "omp": omp_env(),
            "sample": f"reference gg::run (oracle/_ref, OMP threads={cores}) on the same graph, "
                      f"max_iterations={WINDOW_ITERS} ({ALPHA} approximate iterations + 1 superstep, "
                      f"gg scheme); GTEPS = processed_edges / RunReport wall_seconds (sparsify "
                      f"outside); {w['elapsed_s']} s of CPU run incl. serial sparsify"}


def reference_accuracy(wl, g, handle):
    """The reference's own score of its gg run against its accurate run
    (bench.cpp:133-190 protocol: accurate run to convergence within the
    default budget, gg run capped at its iterations)."""
    import numpy as np

    from oracle.oracle import ACCURATE, GG, WCC, BP_EDGE, Reference
    prog, pp = ref_params(wl, g)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    a = Reference.run(g, prog, scheme=ACCURATE, max_iterations=budget_for(wl, g.n), seed=wl["seed"],
                      threads=cores, handle=handle, **pp)
    r = Reference.run(g, prog, scheme=GG, sigma=SIGMA, theta=wl["theta"], alpha=ALPHA,
                      max_iterations=a.iterations_run, seed=wl["seed"], threads=cores, handle=handle,
                      **pp)

    def proj(x):
        x = np.asarray(x)
        if prog == BP_EDGE:
            return x[:, 0].astype(np.float64)
        if prog == WCC:
            return x.astype(np.float64)
        return x.astype(np.float64)
    kind = METRIC_KIND[wl["prog"]]
    k = max(1, g.n // 100)
    err = Reference.metric(kind, proj(r.props), proj(a.props), k)
    return {"metric": METRIC_NAME[kind], "accuracy": round((1.0 - err) * 100.0, 6),
            "k": k if kind == 0 else None,
            "edge_ratio": round(r.total_processed_edges / a.total_processed_edges, 6)
            if a.total_processed_edges else 1.0,
            "accurate_iterations": a.iterations_run, "gg_iterations": r.iterations_run,
            "elapsed_s": round(time.perf_counter() - t0, 1)}


def reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import GG, Reference
    wl = WORKLOADS[args.workload]
    if not Reference.available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libggref.so not built (needs /root/reference)"}))
        return
    t = time.perf_counter()
    g = ref_inputs(wl)
    h = Reference.graph(g)
    log(f"reference inputs n={g.n} e={g.e} in {time.perf_counter() - t:.1f}s")
    prog, pp = ref_params(wl, g)
    cores = os.cpu_count() or 1

    def step():
        r = Reference.run(g, prog, scheme=GG, sigma=SIGMA, theta=wl["theta"], alpha=ALPHA,
                          max_iterations=STEP_ITERS, seed=wl["seed"], threads=cores, handle=h, **pp)
        assert r.status == 0, r.msg
        return r
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    samples = [step() for _ in range(args.steps)]
    elapsed = time.perf_counter() - t0
    edges = sum(r.total_processed_edges for r in samples)
    wall = sum(sum(r.wall_seconds) for r in samples)
    value = round(edges / wall / 1e9, 6) if wall else None
    # beyond the timed steps: per-mode rates over a window with a superstep,
    # the 1-thread rate, and the reference's own accuracy
    window = reference_window(wl, g, handle=h)
    one = reference_one_thread(wl, g)
    acc = reference_accuracy(wl, g, h) if not args.no_accuracy else None
    Reference.free(h)
    cpu = {"value": value, "unit": "GTEPS", "cores": cores, "kind": "reference",
           "sparsified": window["sparsified"], "full": window["full"],
           "window": window, "one_thread": one, "cpu_model": cpu_model(), "omp": omp_env(),
           "sample": f"reference gg::run (oracle/_ref, OMP threads={cores}), gg scheme, each step "
                     f"max_iterations={STEP_ITERS} (the first approximate iteration); GTEPS = "
                     f"processed_edges / RunReport wall_seconds (sparsify outside); window = "
                     f"{WINDOW_ITERS} iterations incl. a superstep, once"}
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed / max(args.steps, 1) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE[wl["prog"]],
        "data": "synthetic R-MAT (seeded, CPU generator)",
        "config": config_json(args, wl, world) | {"vertices": g.n, "edges": g.e},
        "step": {"what": "bounded sample: the first (approximate) iteration of the gg run",
                 "max_iterations": STEP_ITERS, "iterations_per_step": STEP_ITERS},
        "accuracy": acc,
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c5")
    ap.add_argument("--transport", choices=["nccl", "local"], default="nccl")
    ap.add_argument("--no-fused", action="store_true",
                    help="N > 1: all-gather the messages after the vertex kernel instead of the "
                         "fused peer-memory stores")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true", help="reference arm: skip its accuracy runs")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule: W >= 3)")
        args.warmup = 3
    if args.impl == "reference":
        return reference(args)
    if args.transport == "local" and args.gpus > 1:
        return ours_local(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    ours(args)


if __name__ == "__main__":
    main()
