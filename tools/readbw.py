"""HBM read ceiling on this B200 (development aid): python tools/readbw.py"""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libreadbw.so")
if not os.path.exists(SO):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--shared",
                           "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "readbw.cu")])
L = ctypes.CDLL(SO)
L.readbw.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                     ctypes.c_void_p]
nbytes = 8 << 30
buf = torch.ones(nbytes // 2, dtype=torch.bfloat16, device="cuda")
out = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
best = 0
for blocks_per_sm in (1, 2, 4, 8):
    for threads in (256, 512):
        for unroll in (4, 8, 16):
            grid = 148 * blocks_per_sm
            for _ in range(2):
                L.readbw(buf.data_ptr(), nbytes, out.data_ptr(), grid, threads, unroll, s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                L.readbw(buf.data_ptr(), nbytes, out.data_ptr(), grid, threads, unroll, s.cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            gbs = 5 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
            best = max(best, gbs)
            print(f"grid {grid:5d} threads {threads} unroll {unroll:2d}: {gbs:7.0f} GB/s", flush=True)
print(f"best read-only: {best:.0f} GB/s")
# copy reference (read+write), like MEASURED_PEAKS
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
print(f"torch copy (read+write): {10 * 2 * a.numel() * 2 / (e0.elapsed_time(e1) / 1e3) / 1e9:.0f} GB/s")
