"""Small, fixed engine run for ncu captures (one gg run of a BASELINE
workload; the first iterations are approximate, then a superstep)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import SIGMA, ALPHA, WORKLOADS, make_program  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--scheme", default="gg")
a = ap.parse_args()
wl = WORKLOADS[a.workload]
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
prog = make_program(ggb, wl, dg, dg.n)
r = ggb.run(dg, prog, ggb.EngineConfig(a.scheme, SIGMA, wl["theta"], ALPHA, a.iters, wl["seed"]),
            timing=True, device_output=True)
for it in r.per_iteration:
    print(it.mode.name, it.processed_edges, f"{it.kernel_ms:.3f} ms",
          f"{it.algo_bytes / it.kernel_ms / 1e6:.1f} GB/s" if it.kernel_ms else "")
