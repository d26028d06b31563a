"""Diagnostic: look-back statistics of one c5 superstep (needs a library built
with -DGGB_CHAIN_STATS=1, GGB_LIB_PATH pointing at it)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10039_b200 as ggb  # noqa: E402
from bench import ALPHA, SIGMA, WORKLOADS, make_program  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
lib = ctypes.CDLL(os.environ["GGB_LIB_PATH"])
dg = ggb.DeviceGraph.rmat(wl["scale"], wl["ef"], wl["seed"], symmetrize=wl["sym"], weights=wl["weights"])
prog = make_program(ggb, wl, dg, dg.n)
cfg = ggb.EngineConfig("gg", SIGMA, wl["theta"], ALPHA, 5, wl["seed"])
out = (ctypes.c_ulonglong * 8)()
for rep in range(3):
    ggb.run(dg, prog, cfg, device_output=True)
    lib.ggb_debug_chain_stats(out)
    v = list(out)
    print(f"look-backs {v[0]}, sleeps {v[1]} ({v[1] / max(v[0], 1):.2f} per look-back), window advances {v[2]} "
          f"({v[2] / max(v[0], 1):.2f}), no-sleep {v[3]} ({100 * v[3] / max(v[0], 1):.1f}%), >8 sleeps {v[4]}, "
          f">64 sleeps {v[5]}, >4 advances {v[6]}, max rounds {v[7]}")
