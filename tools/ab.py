"""A/B timing of engine variants on one box.

    python tools/ab.py c5 base: GGB_SMEM_HOT_KB=192:hot192 LIB=build/ab_x.so:x ...

Each variant is `ENV=VAL,ENV2=VAL2:label` (or `base:`); LIB=path selects an
alternative libggb.so (GGB_LIB_PATH). Every variant runs in its own process
(environment-driven statics start fresh), builds the workload's graph on the
device and reports, over `--reps` whole gg runs after 3 warm-ups: the median
run time (device-resident graph, no timing events) and, from one extra run
with CUDA-event timing, per-mode edge-kernel ms, vertex ms and rebuild ms.
Variants are interleaved `--rounds` times to average out box drift.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["AB_ROOT"])
import torch
import paper_2104_10039_b200 as ggb
from bench import ALPHA, SIGMA, WORKLOADS, budget_for, make_program
wl = WORKLOADS[os.environ["AB_WL"]]
reps = int(os.environ["AB_REPS"])
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
prog = make_program(ggb, wl, dg, dg.n)
acc = ggb.run(dg, prog, ggb.EngineConfig("accurate", max_iterations=budget_for(wl, dg.n)), device_output=True)
cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, acc.iterations_run, wl["seed"])
for _ in range(3):
    ggb.run(dg, prog, cfg, device_output=True)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    r = ggb.run(dg, prog, cfg, device_output=True)
    ts.append(time.perf_counter() - t0)
ts.sort()
t = ggb.run(dg, prog, cfg, device_output=True, timing=True)
per = {}
for it in t.per_iteration:
    k = it.mode.name
    d = per.setdefault(k, {"n": 0, "edge_ms": 0.0, "vertex_ms": 0.0, "rebuild_ms": 0.0, "edges": 0,
                           "edge_bytes": 0})
    d["n"] += 1; d["edge_ms"] += it.edge_ms; d["vertex_ms"] += it.vertex_ms
    d["rebuild_ms"] += it.rebuild_ms; d["edges"] += it.processed_edges; d["edge_bytes"] += it.edge_bytes
for d in per.values():
    d["gbs"] = round(d["edge_bytes"] / d["edge_ms"] / 1e6, 1) if d["edge_ms"] else None
    for k in ("edge_ms", "vertex_ms", "rebuild_ms"):
        d[k] = round(d[k], 3)
print(json.dumps({"median_ms": round(ts[len(ts) // 2] * 1e3, 3), "min_ms": round(ts[0] * 1e3, 3),
                  "iterations": r.iterations_run, "edges": r.total_processed_edges,
                  "launches": r.kernel_launches, "modes": per}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=1)
    a = ap.parse_args()
    for rnd in range(a.rounds):
        for v in a.variants:
            spec, _, label = v.partition(":")
            env = dict(os.environ, AB_ROOT=ROOT, AB_WL=a.workload, AB_REPS=str(a.reps))
            if spec and spec != "base":
                for kv in spec.split(","):
                    k, _, val = kv.partition("=")
                    if k == "LIB":
                        env["GGB_LIB_PATH"] = os.path.join(ROOT, val)
                    else:
                        env[k] = val
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                               timeout=900)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
            try:
                d = json.loads(line)
            except Exception:
                d = {"error": (r.stderr or r.stdout)[-2000:]}
            d.update(variant=label or spec, spec=spec, workload=a.workload, round=rnd)
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
