import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2104_10039_b200 as ggb
from tests.test_gpu_parity import _exact_graph
from tests.parity import to_graph, device_program, SCHEMES
from oracle.oracle import Oracle, PR, WCC, SSSP
n, e = int(sys.argv[1]), int(sys.argv[2])
g = _exact_graph(n, e, n + e)
for scheme in ("gg", "sms"):
    for prog in (PR, WCC):
        ref = Oracle.run(g, prog, scheme=SCHEMES[scheme], sigma=0.5, theta=0.05, alpha=2, max_iterations=12, seed=e, want_flags=True)
        rep = ggb.run(to_graph(ggb, g), device_program(ggb, prog), ggb.EngineConfig(scheme, 0.5, 0.05, 2, 12, e), want_flags=True)
        pe = [r.processed_edges for r in rep.per_iteration]
        print(scheme, prog, "dev", pe)
        print(scheme, prog, "ref", ref.processed_edges, "mask mism", int(np.count_nonzero(rep.flags != ref.flags)))
        if pe != ref.processed_edges:
            d = np.nonzero(rep.flags != ref.flags)[0]
            print("  first mismatching edges", d[:20], "of", d.size)
