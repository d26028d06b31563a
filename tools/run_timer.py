"""Wall time of back-to-back whole runs (device-resident graph, no timing
events requested) for A/B comparisons: python tools/run_timer.py c2 20"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import ALPHA, SIGMA, WORKLOADS, budget_for, make_program  # noqa: E402

wl = WORKLOADS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
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
print(f"{sys.argv[1]}: iterations {r.iterations_run} launches {r.kernel_launches} "
      f"median {ts[len(ts) // 2] * 1e3:.3f} ms min {ts[0] * 1e3:.3f} ms")
