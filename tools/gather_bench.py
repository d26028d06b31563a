"""Calibration: random 8-byte gather bandwidth on this GPU (see gather_bench.cu)."""
import ctypes
import os
import sys

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgbench.so"))
lib.gbench.restype = ctypes.c_float
lib.gbench.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_uint64, ctypes.c_void_p] + [ctypes.c_int] * 4
N = 1 << 26
E = 922_099_679
dev = torch.device("cuda")
x = torch.rand(N, dtype=torch.float64, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
for name in ("uniform", "rmat"):
    if name == "uniform":
        idx = torch.randint(0, N, (E,), dtype=torch.int32, device=dev)
    else:  # R-MAT source marginal: each of 26 bits is 1 with p = c + d = 0.24
        idx = torch.zeros(E, dtype=torch.int32, device=dev)
        for b in range(26):
            idx |= (torch.rand(E, device=dev) < 0.24).to(torch.int32) << (25 - b)
        idx = idx.sort().values if len(sys.argv) > 1 and sys.argv[1] == "sorted" else idx
    for unroll in (4, 8, 16, 32):
        for threads, occ in ((256, 8), (128, 16)):
            blocks = 148 * occ
            ms = lib.gbench(idx.data_ptr(), x.data_ptr(), E, out.data_ptr(), unroll, blocks, threads, 3)
            gbs = E * 12 / ms / 1e6
            print(f"{name:8s} unroll {unroll:2d} threads {threads} blocks {blocks}: {ms:7.3f} ms "
                  f"{E / ms / 1e6:7.1f} Gedge/s  {gbs:7.1f} GB/s (12 B/edge)", flush=True)
    del idx
