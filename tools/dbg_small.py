"""Quick device sanity run with progress output (small graphs, every scheme)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_10039_b200 as ggb
from oracle.oracle import Oracle
for scale, sym, prog in ((8, False, "pr"), (12, False, "pr"), (12, True, "wcc"), (16, True, "wcc"), (16, False, "pr")):
    g = Oracle.rmat(scale, 16, 3)
    if sym:
        g = Oracle.symmetrized(g)
    graph = ggb.Graph(g.n, g.off, g.src, None, g.outdeg)
    p = ggb.pagerank_spec() if prog == "pr" else ggb.wcc_spec()
    for scheme in ("sp", "sms", "gg"):
        t = time.time()
        print("start", scale, prog, scheme, flush=True)
        r = ggb.run(graph, p, ggb.EngineConfig(scheme, 0.5, 0.01 if prog == "pr" else 0.0, 2, 10, 1))
        print(scale, prog, scheme, r.iterations_run, r.total_processed_edges, f"{time.time()-t:.3f}s", flush=True)
