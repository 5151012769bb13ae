"""Per-rank shard timing on ONE B200: the multi-GPU configs' rank shards run one
at a time on this GPU, so the 1->N strong-scaling of the attention itself can
be read off a single box (gpurun gives one GPU).  Development/evidence aid; the
contract numbers for N > 1 come from `bench.py --gpus N` under torchrun.

  c4: KV-head sharded, rank r owns Hkv/N KV heads and
      their G q-heads for all 512 requests; every rank's work is identical, so
      rank 0's shard is timed.
  c5: the GPU-resident share split by LPT on ctx (paper_2411_01142_b200.shard.
      lpt_assign); every rank's shard is timed and the max is the step time.

The data path has no collective (units are independent), so the per-rank
kernel time is the N-GPU step time up to the (separately reported, overlapped)
head all-gather.  Prints one JSON line per (config, N).

  python tools/shard_time.py [c4] [c5] [--reps 5] [--n 1,2,4,8] [--chunks 128,256,...]

With several --chunks, rank 0's shard of each N is timed at every chunk size
(a tuning sweep; NEO_ATTN_CFG selects the kernel shape).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import WORKLOADS  # noqa: E402
from paper_2411_01142_b200 import neo  # noqa: E402
from paper_2411_01142_b200.shard import head_shard, lpt_assign  # noqa: E402


def time_batch(gb, reps, layers, chunk=0):
    """Median per-layer device time (s) of back-to-back decode_attn calls cycling
    the batch's distinct layer pools (each > L2 or flushed)."""
    chunk = chunk or neo.plan_chunk(gb.ctx, gb.hkv, gb.P)
    ws = neo.make_workspace(gb.B, gb.hq, gb.hkv, gb.max_seq_len, chunk)
    out = torch.empty(gb.B, gb.hq, 128, dtype=torch.bfloat16, device="cuda")
    flush = None
    if gb.layers * gb.kv_bytes_per_call() < 1e9:
        flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()

    def run():
        for l in range(layers):
            k, v = gb.layer(l)
            neo.decode_attn(gb.q[l % gb.layers], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=out,
                            chunk_tokens=chunk, workspace=ws, stream=s,
                            kv_stable=os.environ.get("NEO_KV_STABLE", "1") != "0")

    for _ in range(3):
        if flush is not None:
            flush.sum()
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / layers)
    return float(np.median(ts)), chunk


def sweep(configs, ns, chunks, reps):
    shape = os.environ.get("NEO_ATTN_CFG", "default")
    for name in configs:
        wl = WORKLOADS[name]
        ctx_all = wl.contexts()
        for n in ns:
            if name == "c4":
                kvh, qh = head_shard(wl.hq, wl.hkv, 0, n)
                gb = GpuBatch(wl, ctx=ctx_all, kv_heads=kvh, q_heads=qh)
            else:
                gb = GpuBatch(wl, ctx=ctx_all, req_ids=np.sort(lpt_assign(ctx_all, n)[0]))
            kvb = gb.kv_bytes_per_call()
            row = {}
            for c in chunks:
                t, _ = time_batch(gb, reps, 16, c)
                row[c] = round(kvb / t / 1e9, 0)
            print(json.dumps({"config": name, "n": n, "shape": shape, "kv_gbs_by_chunk": row,
                              "default_chunk": neo.default_chunk(gb.B, gb.hkv, gb.max_seq_len),
                              "planned_chunk": neo.plan_chunk(gb.ctx, gb.hkv, gb.P)}), flush=True)
            del gb
            torch.cuda.empty_cache()


def main():
    # accept --opt=value as well as --opt value
    sys.argv = [sys.argv[0]] + [x for a in sys.argv[1:] for x in (a.split("=", 1) if a.startswith("--") and "=" in a
                                                                   else [a])]
    argv = sys.argv[1:]
    args = [a for i, a in enumerate(argv) if not a.startswith("--") and (i == 0 or not argv[i - 1].startswith("--"))]
    reps = 5
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    configs = args or ["c4", "c5"]
    ns = (1, 2, 4, 8)
    if "--n" in sys.argv:
        ns = tuple(int(x) for x in sys.argv[sys.argv.index("--n") + 1].split(","))
    chunks = [0]
    if "--chunks" in sys.argv:
        chunks = [int(x) for x in sys.argv[sys.argv.index("--chunks") + 1].split(",")]
    if len(chunks) > 1:
        return sweep(configs, ns, chunks, reps)
    for name in configs:
        wl = WORKLOADS[name]
        ctx_all = wl.contexts()
        t1 = None
        for n in ns:
            per_rank = []
            kv_total = 0
            if name == "c4":
                kvh, qh = head_shard(wl.hq, wl.hkv, 0, n)
                gb = GpuBatch(wl, ctx=ctx_all, kv_heads=kvh, q_heads=qh)
                t, chunk = time_batch(gb, reps, 16)
                per_rank = [t] * n                  # identical work on every rank
                kv_total = gb.kv_bytes_per_call() * n
                del gb
            else:
                parts = lpt_assign(ctx_all, n)
                for r in range(n):
                    gb = GpuBatch(wl, ctx=ctx_all, req_ids=np.sort(parts[r]))
                    t, chunk = time_batch(gb, reps, 8)
                    per_rank.append(t)
                    kv_total += gb.kv_bytes_per_call()
                    del gb
                    torch.cuda.empty_cache()
            torch.cuda.empty_cache()
            t_step = max(per_rank)
            if n == 1:
                t1 = t_step
            print(json.dumps({"config": name, "n": n, "per_rank_us": [round(x * 1e6, 1) for x in per_rank],
                              "step_us": round(t_step * 1e6, 1), "kv_gbs_total": round(kv_total / t_step / 1e9, 1),
                              "speedup_vs_1": round(t1 / t_step, 3) if t1 else None, "imbalance": round(t_step / np.mean(per_rank), 4),
                              "chunk": chunk}), flush=True)


if __name__ == "__main__":
    main()
