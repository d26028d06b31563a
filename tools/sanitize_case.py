"""Small engine runs that exercise every lock-free / look-back kernel, for
compute-sanitizer (one tool per invocation):
  superstep chain (edge_chain_kernel: packed {state, value} slots, PageRank;
  edge_kernel<kEdgeChain>: BP with 5 states, release/acquire slots), the
  one-pass scan/compaction and layout look-backs (scan_compact_kernel,
  sp_layout_kernel), the hot-table gather (WCC), the vertex epilogue.
Results are checked against a second, grid-capped run (bit-identical)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402

dg = ggb.DeviceGraph.rmat(12, 16, 7)
sym = dg.symmetrized()
cases = [(dg, ggb.pagerank_spec(), "gg"), (dg, ggb.bp_spec(5, 0.7), "gg"),
         (dg, ggb.bp_spec(2, 0.8), "sms"), (sym, ggb.wcc_spec(), "gg"),
         (dg, ggb.sssp_spec(0, True), "gg")]
for g, prog, scheme in cases:
    cfg = ggb.EngineConfig(scheme, 0.5, 0.05, 2, 12, 3)
    a = ggb.run(g, prog, cfg, want_flags=True)
    b = ggb.run(g, prog, cfg, want_flags=True, grid_ctas=3)
    assert np.array_equal(np.asarray(a.final_properties).view(np.uint8),
                          np.asarray(b.final_properties).view(np.uint8))
    assert np.array_equal(a.flags, b.flags)
    print(type(prog).__name__, scheme, a.iterations_run, "iterations ok")
sym.close()
dg.close()
print("sanitize case ok")
