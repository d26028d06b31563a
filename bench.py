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
  python bench.py --impl reference ...   (reference CPU engine, rank 0 only)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS of full and sparsified gather iterations; % of HBM roofline"
WORKLOADS = {
    "c1": dict(prog="pr", scale=16, ef=16, seed=1, theta=0.01, weights=None, sym=False),
    "c2": dict(prog="sssp", scale=22, ef=16, seed=2, theta=0.05, weights="u32", sym=False),
    "c3": dict(prog="wcc", scale=23, ef=16, seed=3, theta=0.0, weights=None, sym=True),
    "c4": dict(prog="bp", scale=25, ef=16, seed=4, theta=0.01, weights="coupling", sym=False),
    "c5": dict(prog="pr", scale=26, ef=28, seed=5, theta=0.01, weights=None, sym=False),
}
SIGMA, ALPHA = 0.5, 4
DTYPE = {"pr": "f64", "sssp": "u32", "wcc": "u32", "bp": "f32 storage / f64 arithmetic"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_json(args, wl, world):
    return {
        "workload": f"{args.workload}: {wl['prog'].upper()} on R-MAT s{wl['scale']} EF{wl['ef']} "
                    f"seed {wl['seed']}" + (" symmetrised" if wl["sym"] else ""),
        "scale": wl["scale"], "edge_factor": wl["ef"], "seed": wl["seed"],
        "scheme": "gg", "sigma": SIGMA, "theta": wl["theta"], "alpha": ALPHA,
        "rmat_abcd": [0.57, 0.19, 0.19, 0.05], "parallelism": f"dst-partition x{world}",
        "l2": "inputs larger than L2 (CSC >> 126 MB)" if wl["scale"] >= 22
              else "L2-resident graph (no flush: launch-bound parity config)",
    }


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

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
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        os.unlink(self.path)
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


def ours(args):
    import numpy as np
    import torch

    import paper_2104_10039_b200 as ggb

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    exchange = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [ggb.Exchange.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        exchange = ggb.Exchange(rank, world, uid[0])
    wl = WORKLOADS[args.workload]
    t_setup = time.perf_counter()
    dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"],
                              weights=wl["weights"], device=local, rank=rank, nranks=world,
                              exchange=exchange.handle if exchange else None)
    n, e = dg.n, dg.e
    info = dg.info()
    program = make_program(ggb, wl, dg, n)
    acc = ggb.run(dg, program, ggb.EngineConfig("accurate", max_iterations=budget_for(wl, n)),
                  device_output=True)
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
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    reps = [ggb.run(dg, program, cfg, timing=True, device_output=True) for _ in range(args.steps)]
    ev1.record()
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    edges = sum(r.total_processed_edges for r in reps)
    value = edges / (ms / 1e3) / 1e9
    launches = sum(r.kernel_launches for r in reps)

    # per-mode GTEPS and the dominant kernel's roofline (CUDA events on the
    # engine's own stream, recorded around every gather launch)
    per = [it for r in reps for it in r.per_iteration]
    approx = [it for it in per if it.mode == ggb.IterationMode.approximate]
    full = [it for it in per if it.mode != ggb.IterationMode.approximate]
    frac_rank = info["e_local"] / max(e, 1)

    def gteps(its):  # gather step (edge + vertex kernels) of this rank
        t = sum(i.kernel_ms for i in its)
        return (sum(i.processed_edges for i in its) * frac_rank / (t / 1e3) / 1e9) if t else None

    def gbs(its, b="edge_bytes", m="edge_ms"):  # algorithmic bytes / CUDA-event time
        t = sum(getattr(i, m) for i in its)
        return (sum(getattr(i, b) for i in its) / (t / 1e3) / 1e9) if t else None

    peaks = load_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    dom = approx if approx else full  # the dominant kernel: the approximate edge gather
    achieved = gbs(dom)
    traffic, ncu = load_traffic(args.workload)
    roofline = {
        "bound": "hbm", "kernel": "edge_kernel<kEdgePlain> (approximate gather, sparsified CSC)"
        if approx else "edge_kernel (full gather)",
        "achieved": round(achieved, 1) if achieved else None, "peak": peak,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)" if "hbm_gbs" in peaks
        else "fallback 6650 GB/s (B200_PROFILING.md)",
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

    # ---- end to end through the public API: pinned host CSC -> H2D upload
    # (gg_dev_graph_create), run, D2H of the final properties, every step.
    e2e = None
    if not args.no_e2e:
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
    else:
        host = None

    # ---- reference CPU path beside it (rank 0, N=1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if host is None:
            host = dg.to_host()
        cpu = reference_sample(wl, host, n, program_seed=wl["seed"], repeats=1)

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPE[wl["prog"]], "data": "synthetic R-MAT (seeded, built on device)",
        "config": config_json(args, wl, world) | {"vertices": n, "edges": e,
                                                 "max_iterations": budget,
                                                 "iterations_per_step": reps[0].iterations_run,
                                                 "edges_per_step": reps[0].total_processed_edges},
        "gteps_sparsified_kernel": round(gteps(approx), 3) if gteps(approx) else None,
        "gteps_full_kernel": round(gteps(full), 3) if gteps(full) else None,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if exchange:
        dg.close()
        exchange.close()
    if dist:
        dist.destroy_process_group()


# --------------------------------------------------------------------------
# reference arm (the unmodified reference, oracle/_ref/libggref.so)
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


SAMPLE_ITERS = 1


def reference_sample(wl, host_graph, n, program_seed, repeats=1, handle=None, g=None):
    """Bounded sample: the reference gg::run (gg scheme, all host threads)
    capped at SAMPLE_ITERS iteration(s); GTEPS from its own RunReport."""
    from oracle.oracle import GG, Reference
    if not Reference.available():
        return None
    g = g if g is not None else ref_inputs(wl, host_graph)
    prog, pp = ref_params(wl, g)
    own = handle is None
    h = handle if handle is not None else Reference.graph(g)
    cores = os.cpu_count() or 1
    edges = wall = 0
    t0 = time.perf_counter()
    for _ in range(repeats):
        r = Reference.run(g, prog, scheme=GG, sigma=SIGMA, theta=wl["theta"], alpha=ALPHA,
                          max_iterations=SAMPLE_ITERS, seed=program_seed, threads=cores,
                          handle=h, **pp)
        edges += r.total_processed_edges
        wall += sum(r.wall_seconds)
    elapsed = time.perf_counter() - t0
    if own:
        Reference.free(h)
    return {"value": round(edges / wall / 1e9, 5) if wall else None, "unit": "GTEPS",
            "cores": cores, "kind": "reference",
            "sample": f"reference gg::run (oracle/_ref, OMP threads={cores}) on the same graph, "
                      f"max_iterations={SAMPLE_ITERS} (first approximate iteration), x{repeats}; "
                      f"GTEPS = processed_edges / RunReport wall_seconds; "
                      f"{elapsed:.1f}s incl. serial sparsify/setup"}


def reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Reference
    wl = WORKLOADS[args.workload]
    if not Reference.available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libggref.so not built (needs /root/reference)"}))
        return
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    t = time.perf_counter()
    g = ref_inputs(wl)
    h = Reference.graph(g)
    log(f"reference inputs n={g.n} e={g.e} in {time.perf_counter() - t:.1f}s")
    for _ in range(args.warmup):
        reference_sample(wl, None, g.n, wl["seed"], handle=h, g=g)
    t0 = time.perf_counter()
    samples = [reference_sample(wl, None, g.n, wl["seed"], handle=h, g=g)
               for _ in range(args.steps)]
    elapsed = time.perf_counter() - t0
    Reference.free(h)
    vals = [s["value"] for s in samples if s and s["value"]]
    value = statistics.mean(vals) if vals else None
    cpu = dict(samples[0])
    cpu["value"] = value
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed / max(args.steps, 1) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE[wl["prog"]],
        "data": "synthetic R-MAT (seeded, CPU generator)",
        "config": config_json(args, wl, world) | {"vertices": g.n, "edges": g.e},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule: W >= 3)")
        args.warmup = 3
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
