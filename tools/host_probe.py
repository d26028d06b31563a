"""Host-side cost of one gg run: wall time of ggb.run (device_output) vs the
sum of its iteration walls, per workload (small graphs are host-bound)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import SIGMA, ALPHA, WORKLOADS, make_program, budget_for  # noqa: E402

for name in sys.argv[1:]:
    wl = WORKLOADS[name]
    dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
    prog = make_program(ggb, wl, dg, dg.n)
    acc = ggb.run(dg, prog, ggb.EngineConfig("accurate", max_iterations=budget_for(wl, dg.n)),
                  device_output=True)
    cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, acc.iterations_run, wl["seed"])
    for timing in (False, True):
        for _ in range(3):
            ggb.run(dg, prog, cfg, device_output=True, timing=timing)
        ts, iw = [], []
        for _ in range(20):
            t0 = time.perf_counter()
            r = ggb.run(dg, prog, cfg, device_output=True, timing=timing)
            ts.append(time.perf_counter() - t0)
            iw.append(r.total_wall_seconds)
        ts.sort(); iw.sort()
        print(f"{name} timing={timing}: run wall median {ts[10]*1e3:.3f} ms, iterations {iw[10]*1e3:.3f} ms, "
              f"iterations_run {r.iterations_run}, launches {r.kernel_launches}")
