"""Measure NEO's cost-model tables on this B200 box ("offline profiling ...
and linear interpolation") for LLaMa-3.1-8B and write
profiles/cost_profile_b200_llama8b.json:

  lin   linear stage per layer (QKV, O, gate/up, down GEMMs: library cuBLAS via
        torch.matmul -- a cost-table measurement, not part of the hot path)
  gdec  GPU decode attention per layer: our neo_decode_attn (at the planner's chunk)
        over batches of ~1K contexts
  gpre  prefill attention per layer: our neo_prefill_attn (paged, causal, one
        whole prompt of t tokens), fitted to a t^2 + b t
  cdec  CPU decode attention per layer: our neo_cpu_decode_attn on the host cores
  pcie  pinned D2H memcpy bandwidth

python tools/profile_costs.py"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import neo_inputs as ni  # noqa: E402
from neo_inputs.gpu import GpuBatch  # noqa: E402
from neo_inputs.workloads import Workload  # noqa: E402
from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo  # noqa: E402

H, HQ, HKV, D, FF = 4096, 32, 8, 128, 14336


def gpu_time(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def linear_table():
    ws = [torch.randn(H, (HQ + 2 * HKV) * D, dtype=torch.bfloat16, device="cuda"),
          torch.randn(HQ * D, H, dtype=torch.bfloat16, device="cuda"),
          torch.randn(H, 2 * FF, dtype=torch.bfloat16, device="cuda"),
          torch.randn(FF, H, dtype=torch.bfloat16, device="cuda")]
    out = []
    for t in (1, 8, 32, 128, 256, 512, 1024, 2048, 4096, 8192):
        xs = [torch.randn(t, w.shape[0], dtype=torch.bfloat16, device="cuda") for w in ws]

        def layer():
            for x, w in zip(xs, ws):
                torch.matmul(x, w)
        out.append((t, gpu_time(layer)))
    return out


def gdec_table():
    out = []
    for B in (8, 32, 128, 256, 512, 1024):
        wl = Workload("p", "LLaMa-3.1-8B", HQ, HKV, B, 1, 1, "uniform", (1024,), index=50)
        gb = GpuBatch(wl, layers=1)
        k, v = gb.layer(0)
        C = neo.plan_chunk(gb.ctx, HKV, gb.P)           # the a0 planner's choice, as bench.py
        ws = neo.make_workspace(gb.B, HQ, HKV, gb.max_seq_len, C)
        o = torch.empty(gb.B, HQ, D, dtype=torch.bfloat16, device="cuda")
        t = gpu_time(lambda: neo.decode_attn(gb.q[0], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=o,
                                             workspace=ws, chunk_tokens=C))
        out.append((int(gb.ctx.astype(np.int64).sum() + gb.B), t))
        del gb
        torch.cuda.empty_cache()
    return out


def gpre_fit():
    pts = []
    P = 16
    for t in (128, 256, 512, 1024, 2048, 4096):
        npg = (t + P - 1) // P
        kp = torch.randn(npg, HKV, P, D, dtype=torch.bfloat16, device="cuda")
        vp = torch.randn(npg, HKV, P, D, dtype=torch.bfloat16, device="cuda")
        bt = torch.arange(npg, dtype=torch.int32, device="cuda").view(1, -1)
        sl = torch.tensor([t], dtype=torch.int32, device="cuda")
        qo = torch.tensor([0, t], dtype=torch.int32, device="cuda")
        q = torch.randn(t, HQ, D, dtype=torch.bfloat16, device="cuda")
        o = torch.empty_like(q)
        pts.append((t, gpu_time(lambda: neo.prefill_attn(q, kp, vp, bt, sl, qo, t, out=o))))
    ts = np.array([p[0] for p in pts], dtype=np.float64)
    ys = np.array([p[1] for p in pts])
    A = np.stack([ts * ts, ts], axis=1)
    a, b = np.linalg.lstsq(A, ys, rcond=None)[0]
    return max(float(a), 0.0), max(float(b), 0.0), pts


def cdec_table():
    out = []
    P = 16
    nth = len(os.sched_getaffinity(0))
    for B in (4, 16, 64, 256):
        ctx = ni.ctx_uniform(51, B, 1024)
        table, nh = ni.block_tables(51, ctx, P)
        host = np.random.default_rng(0).integers(0x3c00, 0x3f80, size=(nh, 1, 2, HKV, P, D), dtype=np.uint16)
        q = ni.q_bits(51, 0, np.arange(B), HQ, D)
        pool = neo.KVPool(1, HKV, num_gpu_pages=1, num_host_pages=nh, page_size=P, allocate=False, host_array=host)
        pool.cpu_decode_attn(0, q, table, ctx, num_threads=nth)
        t0 = time.time()
        reps = 5
        for _ in range(reps):
            pool.cpu_decode_attn(0, q, table, ctx, num_threads=nth)
        out.append((int(ctx.astype(np.int64).sum() + B), (time.time() - t0) / reps))
    return out, nth


def pcie():
    n = 1 << 30
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    t = gpu_time(lambda: host.copy_(dev, non_blocking=True), reps=5, warm=2)
    return n / t


def main():
    lin = linear_table()
    gdec = gdec_table()
    a, b, pre = gpre_fit()
    cdec, nth = cdec_table()
    bw = pcie()
    prof = {"model": "LLaMa-3.1-8B", "gpu": torch.cuda.get_device_name(), "host_threads": nth,
            "L": 32, "t_prl": 50e-6, "t_pol": 100e-6,
            "lin": lin, "gdec": gdec, "gpre_a": a, "gpre_b": b, "gpre_points": pre, "cdec": cdec,
            "page_size": 16, "max_batch_tokens": 8192, "pcie_bytes_per_s": bw,
            "kv_bytes_per_token_layer": HKV * D * 2 * 2,
            "note": "lin: cuBLAS GEMMs of one LLaMa-3.1-8B layer; gdec: neo_decode_attn; gpre: neo_prefill_attn; "
                    "cdec: neo_cpu_decode_attn; t_prl/t_pol assumed (embedding, LM head)"}
    path = os.environ.get("NEO_PROFILE_OUT") or os.path.join(ROOT, "profiles", "cost_profile_b200_llama8b.json")
    json.dump(prof, open(path, "w"), indent=1)
    print(json.dumps(prof, indent=1))


if __name__ == "__main__":
    main()
