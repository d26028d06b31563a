"""Fraction of gathers (full list, and the sigma = 0.5 sparsified list) whose
message slot lies below 2^k, with slots in the engine's order (out-degree
octave desc, id asc): how much a shared-memory table of the hottest slots
could take."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5")
a = ap.parse_args()
wl = WORKLOADS[a.workload]
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
h = dg.to_host()
deg = np.asarray(h.out_degree, dtype=np.int64)
cls = np.where(deg > 0, np.floor(np.log2(np.maximum(deg, 1))).astype(np.int64) + 1, 0)
order = np.lexsort((np.arange(deg.size), -cls))
slot = np.empty(deg.size, dtype=np.int64)
slot[order] = np.arange(deg.size)
src = np.asarray(h.in_sources)
s = slot[src]
e = s.size
print(f"{a.workload}: E={e}")
for k in (10, 12, 13, 14, 15, 16, 18, 20, 22):
    print(f"  slot < 2^{k:2d} ({(1 << k) * 8 / 1024:8.0f} KB of f64): {np.count_nonzero(s < (1 << k)) / e:.3f}")
