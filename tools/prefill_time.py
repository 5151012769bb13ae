"""Time neo_prefill_attn (causal paged GQA prefill) on synthetic prompts and set
it beside library kernels on the same shapes (torch SDPA, flash_attn varlen when
importable).  TFLOP/s counts the causal algorithmic work: for every q-head and
query row at position p, 4 * D * (p + 1) flops (QK^T and PV, multiply + add).

python tools/prefill_time.py [B] [L] [reps]"""
import itertools
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_01142_b200 import neo  # noqa: E402

HQ, HKV, D, P = 32, 8, 128, 16


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def run_ragged(lens, reps, flush):
    """Whole prompts of the given lengths (bench.py's prefill leg shape)."""
    B = len(lens)
    npg = [(n + P - 1) // P for n in lens]
    k_pages = torch.randn(sum(npg), HKV, P, D, device="cuda", dtype=torch.bfloat16)
    v_pages = torch.randn(sum(npg), HKV, P, D, device="cuda", dtype=torch.bfloat16)
    bt = torch.zeros(B, max(npg), dtype=torch.int32, device="cuda")
    o = 0
    for b, m in enumerate(npg):
        bt[b, :m] = torch.arange(o, o + m, dtype=torch.int32)
        o += m
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    qo = torch.tensor([0] + list(itertools.accumulate(lens)), dtype=torch.int32, device="cuda")
    q = torch.randn(sum(lens), HQ, D, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    buf = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(reps + 3):
        if flush:
            buf.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        neo.prefill_attn(q, k_pages, v_pages, bt, sl, qo, max(lens), out=out)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = sum(ts) / len(ts)
    flops = sum(4.0 * D * HQ * n * (n + 1) / 2 for n in lens)
    print(f"ragged {lens} flush={flush}: {t * 1e6:.1f} us {flops / t / 1e12:.1f} TF/s")


def run(B, L, reps):
    npg = (L + P - 1) // P
    k_pages = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
    v_pages = torch.randn(B * npg, HKV, P, D, device="cuda", dtype=torch.bfloat16)
    perm = torch.randperm(B * npg, device="cuda").to(torch.int32)
    bt = perm.view(B, npg).contiguous()
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    qo = torch.arange(0, (B + 1) * L, L, dtype=torch.int32, device="cuda")
    q = torch.randn(B * L, HQ, D, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    flops = 4.0 * D * HQ * B * L * (L + 1) / 2
    t = timed(lambda: neo.prefill_attn(q, k_pages, v_pages, bt, sl, qo, L, out=out), reps)
    res = {"neo": t}
    # library references on contiguous K/V (no paging)
    qs = q.view(B, L, HQ, D).transpose(1, 2)
    ks = torch.randn(B, HKV, L, D, device="cuda", dtype=torch.bfloat16)
    vs = torch.randn(B, HKV, L, D, device="cuda", dtype=torch.bfloat16)
    try:
        res["sdpa"] = timed(lambda: torch.nn.functional.scaled_dot_product_attention(qs, ks, vs, is_causal=True,
                                                                                     enable_gqa=True), reps)
    except Exception as e:  # noqa: BLE001
        print("sdpa failed:", e)
    try:
        from flash_attn import flash_attn_varlen_func
        kf = torch.randn(B * L, HKV, D, device="cuda", dtype=torch.bfloat16)
        vf = torch.randn(B * L, HKV, D, device="cuda", dtype=torch.bfloat16)
        res["flash_attn2"] = timed(lambda: flash_attn_varlen_func(q, kf, vf, qo, qo, L, L, causal=True), reps)
    except Exception as e:  # noqa: BLE001
        print("flash_attn unavailable:", type(e).__name__, str(e)[:100])
    line = " ".join(f"{k} {v * 1e6:8.1f} us {flops / v / 1e12:6.1f} TF/s" for k, v in res.items())
    print(f"B={B:3d} L={L:6d}  {line}")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "ragged":
        import numpy as np
        rng = np.random.default_rng(0x4E454F)
        lens = []
        while True:
            n = int(rng.integers(900, 1101))
            if sum(lens) + n > 8192:
                break
            lens.append(n)
        for flush in (False, True):
            run_ragged(lens, 20, flush)
            run_ragged([1024] * 8, 20, flush)
        return
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    if len(sys.argv) > 2:
        run(int(sys.argv[1]), int(sys.argv[2]), reps)
        return
    for B, L in ((8, 1024), (16, 512), (4, 2048), (2, 4096), (1, 8192), (1, 16384), (64, 128)):
        run(B, L, reps)


if __name__ == "__main__":
    main()
