"""Per-step timeline of one prefill CTA from a trace build of libneo
(-DNEO_PREFILL_TRACE, tools/build_trace.sh -> tools/libneo_trace.so): clock64
stamps in the softmax warps (0 wait start, 1 S ready, 2 S loaded, 3 P stored)
and the MMA warp (4 wait p_full, 5 p_full seen, 6 PV + next S issued).

NEO_LIB=tools/libneo_trace.so python tools/prefill_trace.py [L] [B]
Rows are per-tile running steps of CTA 0 across its items; '*' marks an item's first step."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_01142_b200 import neo  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
HQ, HKV, D, P = 32, 8, 128, 16
npg = L // P
kp = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
vp = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
bt = torch.arange(B * npg, dtype=torch.int32, device="cuda").view(B, npg)
sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
qo = torch.arange(0, (B + 1) * L, L, dtype=torch.int32, device="cuda")
q = torch.randn(B * L, HQ, D, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    neo.prefill_attn(q, kp, vp, bt, sl, qo, L)
torch.cuda.synchronize()
lib = neo.lib()
lib.neo_prefill_trace_ptr.restype = ctypes.c_void_p
ptr = lib.neo_prefill_trace_ptr()
buf = torch.empty(2 * 64 * 16, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
import cuda.bindings.runtime as rt  # noqa: E402
rt.cudaMemcpy(buf.data_ptr(), ptr, buf.numel() * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
tr = buf.cpu().numpy().reshape(2, 64, 16)
t0 = tr[tr > 0].min()
if tr[0, 63, 13]:
    e = tr[0, 63]
    print(f"stream kernel prologue: entry -> PDL wait done {e[14] - e[13]}, -> schedule built {e[15] - e[14]} cycles; "
          f"first S ready {tr[0, 0, 1] - e[13]} after entry; last store issued {tr[1, 63, 13] - e[13]} after entry")
print("step  tile | wait->S ready  ldS  softmax  | MMA: wait p  issue | period")
for j in range(64):
    for t in range(2):
        r = tr[t, j]
        if j == 63 and tr[0, 63, 13]:
            continue
        if r[0] == 0:
            continue
        per = tr[t, j + 1, 1] - r[1] if j + 1 < 64 and tr[t, j + 1, 1] else 0
        mark = "*" if r[7] else " "
        print(f"{j:4d}{mark}{t:4d} | {r[1]-r[0]:8d} {r[2]-r[1]:6d} {r[3]-r[2]:8d} | {r[5]-r[4] if r[4] else 0:8d} "
              f"{r[6]-r[5] if r[6] else 0:6d} | {per:6d}   S@{r[1]-t0}"
              + (f"  epi: P->wait {r[8]-r[3]} o_done {r[9]-r[8]} store {r[10]-r[9]}" if r[8] else "")
              + (f"  next-wait {tr[t, j + 1, 0] - r[10]} (loop top {tr[t, j + 1, 12] - r[10]}, make_item "
                 f"{tr[t, j + 1, 11] - tr[t, j + 1, 12]})" if r[10] and j + 1 < 64 and tr[t, j + 1, 0] else ""))
