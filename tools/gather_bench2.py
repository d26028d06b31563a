"""Calibration 2: does a hot-first slot permutation (R-MAT popularity order:
(popcount(id), id) ascending) raise the random-gather rate?"""
import ctypes
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgbench.so"))
lib.gbench.restype = ctypes.c_float
lib.gbench.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_uint64, ctypes.c_void_p] + [ctypes.c_int] * 4
N = 1 << 26
E = 922_099_679
dev = torch.device("cuda")
x = torch.rand(N, dtype=torch.float64, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
idx = torch.zeros(E, dtype=torch.int32, device=dev)
for b in range(26):
    idx |= (torch.rand(E, device=dev) < 0.24).to(torch.int32) << (25 - b)
ids = torch.arange(N, dtype=torch.int64, device=dev)
pc = torch.zeros(N, dtype=torch.int64, device=dev)
for b in range(26):
    pc += (ids >> b) & 1
order = torch.argsort(pc * N + ids)           # slot -> id
pi = torch.empty(N, dtype=torch.int32, device=dev)
pi[order] = torch.arange(N, dtype=torch.int32, device=dev)  # id -> slot
idx2 = pi[idx.long()]
counts = torch.bincount(idx2.long(), minlength=N).cumsum(0).double() / E
for mb in (32, 64, 100, 126):
    k = mb * (1 << 20) // 8
    print(f"hottest {mb} MB of slots cover {counts[k - 1].item() * 100:.1f}% of gathers")
for name, ix in (("rmat-id", idx), ("rmat-slot", idx2)):
    for unroll, threads, occ in ((16, 128, 16), (32, 128, 16)):
        ms = lib.gbench(ix.data_ptr(), x.data_ptr(), E, out.data_ptr(), unroll, 148 * occ, threads, 3)
        print(f"{name:10s} unroll {unroll}: {ms:7.3f} ms {E / ms / 1e6:7.1f} Gedge/s {E * 12 / ms / 1e6:7.1f} GB/s", flush=True)
