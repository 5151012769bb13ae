import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from harness import PrefillCase, within_tol
import neo_inputs as ni
for ctx, hq in (([128],64), ([1,7,64,65,128,300,1000],64), ([128, 128],64), ([112],64), ([256],64), ([128],32)):
    c = PrefillCase(ctx, ctx, hq, 8, seed=100+hq+8)
    out = c.run()
    got = ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))
    for b in range(c.B):
        ref = c.oracle(b); g = got[c.rows(b)]
        err = np.abs(g-ref)/(2e-3+1e-2*np.abs(ref))
        bad = np.argwhere(err > 1)
        print(ctx, hq, 'b', b, 'worst', float(err.max()), 'nbad', len(bad), 'rows', sorted(set(bad[:,0].tolist()))[:20], 'heads', sorted(set(bad[:,1].tolist()))[:10])
