"""Time neo_cpu_decode_attn (NEXT-2) on this host:
    python tools/cpu_attn_time.py [n_req] [ctx] [threads...]
NEO_CPU_SEQ=1 lays the request's pages out in order (sequential host block
table) instead of the random page ids of a fragmented CPU-cache."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import neo_inputs as ni  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
l = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
threads = [int(x) for x in sys.argv[3:]] or [0]
hq, hkv, P = 32, 8, 16
ctx = ni.ctx_uniform(1, B, l)
table, nh = ni.block_tables(1, ctx, P)
if os.environ.get("NEO_CPU_SEQ") == "1":       # pages of each request contiguous and in order
    o = 0
    for b in range(B):
        n = (int(ctx[b]) + P - 1) // P
        table[b, :n] = np.arange(o, o + n)
        o += n
host = np.zeros((nh, 1, 2, hkv, P, 128), dtype=np.uint16)
rng = np.random.default_rng(0)
host[...] = rng.integers(0x3c00, 0x3f80, size=host.shape, dtype=np.uint16)
q = ni.q_bits(1, 0, np.arange(B), hq, 128)
pool = neo.KVPool(1, hkv, num_gpu_pages=1, num_host_pages=nh, page_size=P, allocate=False, host_array=host)
kvb = int(ctx.sum()) * hkv * 128 * 2 * 2
for th in threads:
    pool.cpu_decode_attn(0, q, table, ctx, num_threads=th)
    t0 = time.time()
    reps = 5
    for _ in range(reps):
        pool.cpu_decode_attn(0, q, table, ctx, num_threads=th)
    dt = (time.time() - t0) / reps
    print(f"threads={th or os.cpu_count()}: {dt * 1e3:.2f} ms, {kvb / dt / 1e9:.2f} GB/s KV, "
          f"{int(ctx.sum()) / dt / 1e6:.1f} M tok/s")
