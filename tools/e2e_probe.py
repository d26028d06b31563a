"""Breakdown of the end-to-end path (upload / run / close) for one workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import ALPHA, SIGMA, WORKLOADS, make_program  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])


def pinned(count, dt):
    return torch.empty(int(count) * np.dtype(dt).itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(dt)


t = time.perf_counter()
host = dg.to_host(alloc=pinned)
print(f"to_host {time.perf_counter() - t:.3f}s")
prog = make_program(ggb, wl, dg, dg.n)
cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, 7, wl["seed"])
dg.close()
shape = {"pr": (dg.n,), "sssp": (dg.n,), "wcc": (dg.n,), "bp": (dg.n, 2)}[wl["prog"]]
out_buf = pinned(int(np.prod(shape)), np.uint32 if wl["prog"] == "wcc" else np.float64).reshape(shape)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g2 = ggb.DeviceGraph.upload(host)
    t1 = time.perf_counter()
    r = ggb.run(g2, prog, cfg, out=out_buf)
    t2 = time.perf_counter()
    g2.close()
    t3 = time.perf_counter()
    print(f"step {i}: upload {t1 - t0:.3f}s run {t2 - t1:.3f}s (engine wall {r.total_wall_seconds:.3f}s) close {t3 - t2:.3f}s")
