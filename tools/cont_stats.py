"""How much of a list superstep pass 2 re-walks: edges of each task's first
vertex when that vertex began in an earlier task (single GPU, pad 0)."""
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
off = np.asarray(h.in_offsets, dtype=np.int64)
e = int(off[-1])
T = 512
ntasks = (e + T - 1) // T
starts = np.arange(ntasks, dtype=np.int64) * T
v = np.searchsorted(off, starts, side="right") - 1       # vertex holding position starts[t]
cont = off[v] < starts
ends = np.minimum(off[v + 1], starts + T)
walked = np.where(cont, ends - starts, 0)
deg = np.diff(off)
print(f"{a.workload}: E={e} tasks={ntasks} cont tasks={int(cont.sum())} ({cont.mean():.3f}) "
      f"pass2 edges={int(walked.sum())} ({walked.sum() / e:.3f} of E)")
for lim in (512, 4096, 65536):
    big = deg > lim
    print(f"  vertices with in-degree > {lim}: {int(big.sum())}, edges {deg[big].sum() / e:.3f} of E")
print(f"  max in-degree {int(deg.max())}")
