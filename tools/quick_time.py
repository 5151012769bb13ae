"""Quick device timing of neo_decode_attn on a workload (development aid; the
contract bench is bench.py).  Usage: python tools/quick_time.py c2 [chunk ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import WORKLOADS  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    chunks = [int(x) for x in sys.argv[2:]] or [-1]      # -1: the a0 planner's chunk (as bench.py)
    wl = WORKLOADS[name]
    t0 = time.time()
    gb = GpuBatch(wl)
    torch.cuda.synchronize()
    print(f"{name}: built {gb.layers} layers, B={gb.B}, sum ctx={int(gb.ctx.sum())} in {time.time() - t0:.1f}s",
          flush=True)
    kvb = gb.kv_bytes_per_call()
    out = torch.empty(gb.B, wl.hq, 128, dtype=torch.bfloat16, device="cuda")
    for C in chunks:
        if C < 0:
            C = neo.plan_chunk(gb.ctx, gb.hkv, gb.P)
        ws = neo.make_workspace(gb.B, wl.hq, wl.hkv, gb.max_seq_len, C)
        L = max(gb.layers, 8)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
        for rep in range(3):
            ev[0].record()
            for l in range(L):
                k, v = gb.layer(l)
                neo.decode_attn(gb.q[l % gb.layers], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=out,
                                chunk_tokens=C, workspace=ws)
                ev[l + 1].record()
            torch.cuda.synchronize()
        ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(L)]
        avg = sum(ts) / L
        print(f"  C={C or neo.default_chunk(gb.B, wl.hkv, gb.max_seq_len)}: avg {avg * 1e3:.1f} us/layer, "
              f"KV {kvb / avg / 1e6:.0f} GB/s  (min {min(ts) * 1e3:.1f} max {max(ts) * 1e3:.1f})", flush=True)


if __name__ == "__main__":
    main()
