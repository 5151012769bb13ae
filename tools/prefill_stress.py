"""Stress: many back-to-back launches of the stream prefill kernel on varied shapes (hang check)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01142_b200 import neo
HQ, HKV, D, P = 32, 8, 128, 16
def case(B, L):
    npg = (L + P - 1) // P
    kp = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
    bt = torch.randperm(B * npg, device="cuda").to(torch.int32).view(B, npg).contiguous()
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    qo = torch.arange(0, (B + 1) * L, L, dtype=torch.int32, device="cuda")
    q = torch.randn(B * L, HQ, D, device="cuda", dtype=torch.bfloat16)
    return lambda: neo.prefill_attn(q, kp, vp, bt, sl, qo, L)
for (B, L, n) in ((8, 1024, 3000), (2, 4096, 500), (37, 300, 2000), (1, 16384, 100), (3, 777, 2000)):
    f = case(B, L)
    t = time.time()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    print(B, L, n, "ok", round(time.time() - t, 2), flush=True)
