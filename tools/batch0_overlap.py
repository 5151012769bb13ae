"""NEO batch-0 on one B200: decode attention of the GPU-resident requests (c2,
one layer: 256 requests x ~1K tokens, HBM-bound) and prefill attention of the
admitted prompts (8 x ~1000 tokens, tensor-bound), run back to back on one
stream vs concurrently on two streams with the persistent prefill grid capped
to N SMs (NEO_PREFILL_CTAS) so decode CTAs take the rest.

python tools/batch0_overlap.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import WORKLOADS  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402

gb = GpuBatch(WORKLOADS["c2"], layers=1)
k, v = gb.layer(0)
ws = neo.make_workspace(gb.B, gb.hq, gb.hkv, gb.max_seq_len)
dout = torch.empty(gb.B, gb.hq, 128, dtype=torch.bfloat16, device="cuda")

rng = np.random.default_rng(0x4E454F)
lens = []
while True:
    n = int(rng.integers(900, 1101))
    if sum(lens) + n > 8192:
        break
    lens.append(n)
P, HQ, HKV, D = 16, 32, 8, 128
npg = [(n + P - 1) // P for n in lens]
kp = torch.randn(sum(npg), HKV, P, D, device="cuda", dtype=torch.bfloat16)
vp = torch.randn(sum(npg), HKV, P, D, device="cuda", dtype=torch.bfloat16)
bt = torch.zeros(len(lens), max(npg), dtype=torch.int32, device="cuda")
o = 0
for b, m in enumerate(npg):
    bt[b, :m] = torch.arange(o, o + m, dtype=torch.int32)
    o += m
sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
qo = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
q = torch.randn(sum(lens), HQ, D, device="cuda", dtype=torch.bfloat16)
pout = torch.empty_like(q)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")


def dec(stream):
    neo.decode_attn(gb.q[0], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=dout, workspace=ws, stream=stream)


def pre(stream):
    neo.prefill_attn(q, kp, vp, bt, sl, qo, max(lens), out=pout, stream=stream)


def timed(fn, reps=10):
    ts = []
    for r in range(reps + 3):
        flush.sum()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


cur = torch.cuda.current_stream()
t_dec = timed(lambda: dec(cur))
t_pre = timed(lambda: pre(cur))
t_seq = timed(lambda: (dec(cur), pre(cur)))
print(f"decode alone {t_dec:.1f} us, prefill alone {t_pre:.1f} us, back to back {t_seq:.1f} us")


def conc():
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        pre(s1)
    with torch.cuda.stream(s2):
        dec(s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for n in (148, 128, 111, 96, 74, 60, 48):
    os.environ["NEO_PREFILL_CTAS"] = str(n)
    t_pre_n = timed(lambda: pre(cur))
    t_c = timed(conc)
    print(f"prefill on {n:3d} SMs: alone {t_pre_n:.1f} us; concurrent with decode {t_c:.1f} us "
          f"({100 * (1 - t_c / t_seq):+.1f} % vs back to back)")
os.environ.pop("NEO_PREFILL_CTAS")
