"""One decode layer of NEO's GPU sub-batch (c2 / c3 / c5 shapes): RoPE + KV append
+ attention as two launches (neo_rope_append -> neo_decode_attn, PDL-chained)
vs one (neo_decode_attn_append), vs attention alone; L2 flushed between reps.

python tools/decode_step_time.py [c2|c3|c5]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import WORKLOADS  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gb = GpuBatch(WORKLOADS[cfg], layers=1)
k, v = gb.layer(0)
C = int(sys.argv[2]) if len(sys.argv) > 2 else neo.plan_chunk(gb.ctx, gb.hkv, gb.P)   # the a0 planner's choice
ws = neo.make_workspace(gb.B, gb.hq, gb.hkv, gb.max_seq_len, C)
out = torch.empty(gb.B, gb.hq, 128, dtype=torch.bfloat16, device="cuda")
kn = torch.randn(gb.B, gb.hkv, 128, dtype=torch.bfloat16, device="cuda")
vn = torch.randn(gb.B, gb.hkv, 128, dtype=torch.bfloat16, device="cuda")
inv = (500000.0 ** (-torch.arange(0, 128, 2, dtype=torch.float64) / 128)).float().cuda()
q = gb.q[0].clone()
flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")


def attn():
    neo.decode_attn(q, k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=out, workspace=ws, chunk_tokens=C)


def separate():
    neo.rope_append(q, inv, k, v, gb.block_table, gb.seq_lens, kn, vn)
    attn()


def fused():
    neo.decode_attn_append(q, k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, kn, vn, inv_freq=inv, out=out,
                           workspace=ws, chunk_tokens=C)


def timed(fn, reps=20):
    ts = []
    for r in range(reps + 3):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


kvb = gb.kv_bytes_per_call()
for name, fn in (("attention only", attn), ("rope_append + attention", separate), ("fused (one launch)", fused)):
    t = timed(fn)
    print(f"{cfg} C={C} {name:26s} {t:8.1f} us   {kvb / t / 1e3:7.1f} GB/s of KV")
