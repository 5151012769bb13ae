import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import neo_inputs as ni
from harness import PrefillCase, within_tol
ctx = [int(x) for x in sys.argv[1].split(",")]
case = PrefillCase(ctx, ctx, 32, 8, seed=1)
out = case.run()
torch.cuda.synchronize()
got = ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))
worst = 0
for b in range(case.B):
    ok, ratio = within_tol(got[case.rows(b)], case.oracle(b))
    worst = max(worst, ratio)
print("done", ctx, "worst err/tol", round(worst, 3))
