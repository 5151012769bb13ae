"""Experiment: does the CTA dispatch order matter?  Times a shard with its
requests in generated order, ascending and descending length order (the
in-order CTA dispatch then approximates LPT or anti-LPT).  Development aid.

  python tools/order_probe.py c4:8 c2s:1 --chunks -2048,-1024,384
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import WORKLOADS  # noqa: E402
from paper_2411_01142_b200.shard import head_shard, lpt_assign  # noqa: E402
from shard_time import time_batch  # noqa: E402

chunks = [int(x) for x in sys.argv[sys.argv.index("--chunks") + 1].split(",")]
for spec in [a for a in sys.argv[1:] if ":" in a]:
    name, n = spec.split(":")
    n = int(n)
    wl = WORKLOADS[name]
    ctx = wl.contexts()
    ids = np.sort(lpt_assign(ctx, n)[0]) if name != "c4" else np.arange(len(ctx))
    kvh, qh = head_shard(wl.hq, wl.hkv, 0, n) if name == "c4" else (None, None)
    for order in ("gen", "asc", "desc"):
        o = ids if order == "gen" else ids[np.argsort(ctx[ids], kind="stable")]
        if order == "desc":
            o = o[::-1]
        gb = GpuBatch(wl, ctx=ctx, req_ids=o, kv_heads=kvh, q_heads=qh, layers=min(wl.layers_built, 8))
        row = {}
        for c in chunks:
            t, _ = time_batch(gb, 5, 16, c)
            row[c] = round(t * 1e6, 1)
        print(json.dumps({"config": name, "n": n, "order": order, "us_by_chunk": row,
                          "gbs_by_chunk": {c: round(gb.kv_bytes_per_call() / (row[c] * 1e-6) / 1e9) for c in row}}),
              flush=True)
        del gb
        torch.cuda.empty_cache()
