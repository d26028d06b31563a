"""Rows (vertices with in-edges) of a BASELINE workload's graph: the
positions the vertex kernel walks after t = 1 (X1)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_10039_b200 as ggb
from bench import WORKLOADS
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
h = dg.to_host()
deg = np.diff(h.in_offsets.astype(np.int64))
print(json.dumps({"n": int(dg.n), "rows": int(np.count_nonzero(deg)),
                  "out_degree_gt0": int(np.count_nonzero(h.out_degree))}))
