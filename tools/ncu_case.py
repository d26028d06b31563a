"""Small, fixed engine run for timing / ncu captures (one gg run of a
BASELINE workload; the first iterations are approximate, then a superstep)."""
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
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
prog = make_program(ggb, wl, dg, dg.n)
for _ in range(a.repeat):
    r = ggb.run(dg, prog, ggb.EngineConfig(a.scheme, SIGMA, wl["theta"], ALPHA, a.iters, wl["seed"]),
                timing=True, device_output=True)
print(f"{a.workload}: run wall {r.total_wall_seconds * 1e3:.2f} ms, {r.kernel_launches} launches")
for it in r.per_iteration:
    gb = lambda b, ms: f"{b / ms / 1e6:7.1f} GB/s" if ms else "      -"
    print(f"{it.mode.name:11s} E={it.processed_edges:11d} edge {it.edge_ms:7.3f} ms {gb(it.edge_bytes, it.edge_ms)} "
          f"| vertex {it.vertex_ms:6.3f} ms {gb(it.vertex_bytes, it.vertex_ms)} | rebuild {it.rebuild_ms:6.3f} "
          f"| wall {it.wall_seconds * 1e3:7.3f} ms")
