"""Subprocess body of test_prefill_slow_epilogue_one_step_items (tests/test_gpu_prefill.py):
runs the stream prefill kernel with a deliberately slow epilogue and checks parity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import neo_inputs as ni  # noqa: E402
from harness import PrefillCase, within_tol  # noqa: E402

ctx = [int(x) for x in sys.argv[1].split(",")]
case = PrefillCase(ctx, ctx, 32, 8, seed=990)
out = case.run()
torch.cuda.synchronize()
got = ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))
for b in range(case.B):
    ok, ratio = within_tol(got[case.rows(b)], case.oracle(b))
    assert ok, f"b={b} err/tol={ratio:.3f}"
print("ok")
