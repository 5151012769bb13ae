"""Small prefill cases for compute-sanitizer (memcheck / racecheck / synccheck):
ragged requests incl. an empty one and a chunk after a prefix, page tails NaN,
RoPE store first (the PDL-chained pair), then prefill attention.

compute-sanitizer --tool racecheck python tools/sanitize_prefill.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import PrefillCase  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402

case = PrefillCase([300, 77, 129, 1], [300, 40, 0, 1], 32, 8, seed=7)
kn = torch.randn(case.T, 8, 128, device="cuda", dtype=torch.bfloat16)
vn = torch.randn(case.T, 8, 128, device="cuda", dtype=torch.bfloat16)
inv = (500000.0 ** (-torch.arange(0, 128, 2, dtype=torch.float64) / 128)).float().cuda()
q = case.qp_dev.clone()
neo.prefill_append(case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.qo_dev, kn, vn, q=q, inv_freq=inv)
out = neo.prefill_attn(q, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.qo_dev, case.max_q_len)
torch.cuda.synchronize()
assert torch.isfinite(out.float()).all()
print("ok", float(out.float().abs().mean()))
