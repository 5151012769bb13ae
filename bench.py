#!/usr/bin/env python
"""bench.py -- NEO's GPU hot path on B200: batched paged GQA decode attention
(+ KV page swap for c3) over synthetic LLaMa-shaped batches.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl neo|reference]

One STEP = one decode iteration's attention for the whole model: one
neo_decode_attn call per layer ("the GPU attention kernel is only invoked
once per iteration" per layer), over the workload's batch, every layer reading
its own KV pool (inputs >> 126 MB L2, so no flush is needed).

Prints ONE JSON line (rank 0).  value = KV bytes read by all ranks / max-over-
ranks device time, in GB/s (BASELINE.json metric); attended tokens/s rides
along.  --impl reference times the fp64 CPU oracle on this box's host cores on a
bounded sample of the same workload (no reference implementation exists; see
DESIGN.md "Reference arm").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention KV GB/s (% of B200 HBM peak) and attended tokens/s @1/2/4/8 GPUs"
NOMINAL_HBM_GBS = 8184.0          # 3996 MHz x 2 x 8192 bit / 8
FALLBACK_HBM_GBS = 6650.0         # B200_PROFILING.md fallback


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c3", help="c1..c5 (BASELINE.json configs), c2s = skewed c2; default c3 "
                   "(batch 128, 4K-8K contexts, the north star's regime, with the swap leg)")
    p.add_argument("--impl", default="neo", choices=["neo", "reference"])
    p.add_argument("--chunk", type=int, default=0, help="split-K chunk tokens (0 = library default)")
    p.add_argument("--fraction", type=float, default=1.0, help="c5: GPU-resident fraction f")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-swap", action="store_true", help="c3: skip the concurrent swap-out")
    p.add_argument("--no-prefill", action="store_true", help="skip the NEXT-3 prefill leg")
    p.add_argument("--graph", action="store_true", help="capture the step's launches in a CUDA graph")
    p.add_argument("--no-kv-stable", action="store_true",
                   help="plain neo_decode_attn (no NEO_ATTN_KV_STABLE early KV prefetch before the PDL wait)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[5 + i] and "Not" not in r[5 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------- setup


def shard_plan(wl, rank, world, fraction):
    """(ctx_all, req_ids, kv_heads, q_heads, scaling, parallelism) for this rank."""
    from paper_2411_01142_b200.shard import head_shard, lpt_assign
    import neo_inputs as ni
    if wl.name == "c4":                                   # tensor parallel by KV head
        kvh, qh = head_shard(wl.hq, wl.hkv, rank, world)
        return wl.contexts(), None, kvh, qh, "strong", f"tp{world} (kv-head sharded)"
    if wl.name == "c5":                                   # GPU-resident share split by LPT (strong)
        ctx = wl.contexts()
        n_gpu = int(round(fraction * len(ctx)))
        resident = np.arange(n_gpu)                       # first f*1024 by id
        parts = lpt_assign(ctx[resident], world)
        return ctx, resident[parts[rank]], None, None, "strong", f"dp{world} (LPT by request)"
    # c1, c2, c3: weak scaling -- every rank serves its own full batch of distinct requests
    if world == 1:
        return wl.contexts(), None, None, None, "weak", "dp1"
    k, a = wl.ctx_kind, wl.ctx_args
    n = wl.batch * world
    if k == "fixed":
        ctx = np.full(n, a[0], dtype=np.int32)
    elif k == "uniform":
        ctx = ni.ctx_uniform(wl.seed, n, a[0])
    elif k == "range":
        ctx = ni.ctx_range(wl.seed, n, a[0], a[1])
    elif k == "lognormal":
        ctx = ni.ctx_lognormal(wl.seed, n, *a)
    else:
        ctx = ni.ctx_loguniform(wl.seed, n, *a)
    return ctx, np.arange(rank * wl.batch, (rank + 1) * wl.batch), None, None, "weak", f"dp{world} (by request)"


def batch_total(wl, gb, world, fraction, ctx_all):
    """Requests served per step over all ranks."""
    if wl.name == "c4":
        return int(gb.B)                        # head-sharded: every rank serves the whole batch
    if wl.name == "c5":
        return int(round(fraction * len(ctx_all)))
    return int(gb.B * world)                    # weak scaling: one batch per rank


def layers_per_step(wl):
    """c1 is a single-layer latency config; the others run every layer of the model."""
    return 1 if wl.name == "c1" else wl.num_layers


# ------------------------------------------------------- multi-rank harness


def aggregate_ranks(t_local_s, kv_local, tok_local, steps, world, head_sharded, dist=None, device="cpu"):
    """Combine per-rank results: time = MAX over ranks, KV bytes =
    SUM; attended tokens SUM for request sharding, but with KV-head sharding
    every rank serves every (request, token, layer) for its own heads, so the
    tokens are counted once (the rank-local count, equal on all ranks).
    Returns (t_max_s, kv_total, tok_total, per_rank_ms_per_step or None)."""
    import torch
    t = torch.tensor([float(t_local_s)], dtype=torch.float64, device=device)
    kv = torch.tensor([float(kv_local)], dtype=torch.float64, device=device)
    tok = torch.tensor([float(tok_local)], dtype=torch.float64, device=device)
    per_rank = None
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [float(x.item()) * 1e3 / steps for x in allt]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(kv, op=dist.ReduceOp.SUM)
        if not head_sharded:
            dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    return float(t.item()), float(kv.item()), float(tok.item()), per_rank


def rank_imbalance(per_rank):
    """Slowest rank over the mean rank (1.0 = balanced)."""
    return round(max(per_rank) / (sum(per_rank) / len(per_rank)), 4)


def reassemble_heads_into(full_l, gathered_l):
    """a9: ``gathered_l`` [world][B][Hq/N][D] (all_gather_into_tensor of the
    head shards, rank-major) -> ``full_l`` [B][Hq][D]: rank r's q heads are
    [r·Hq/N, (r+1)·Hq/N) (shard.head_shard)."""
    world, B, hl, D = gathered_l.shape
    full_l.view(B, world, hl, D).copy_(gathered_l.permute(1, 0, 2, 3))
    return full_l


READBW_SO = os.path.join(ROOT, "tools", "libreadbw.so")
COLL_DEV = "cuda"      # device of the bench's own collective tensors ("cpu" under the gloo harness check)


def build_readbw():
    """Compile the HBM read-ceiling probe (a measurement tool, not the product)."""
    src = os.path.join(ROOT, "tools", "readbw.cu")
    if not os.path.exists(READBW_SO) or os.path.getmtime(READBW_SO) < os.path.getmtime(src):
        tmp = READBW_SO + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--shared",
                               "-Xcompiler", "-fPIC", "-o", tmp, src])
        os.replace(tmp, READBW_SO)
    return READBW_SO


def measure_read_ceiling(gb, stream):
    """This box's HBM read ceiling, measured in the run: a pure streaming read of
    4 GiB of the KV pool (best of 5) -- the denominator a read-only kernel can
    actually reach, reported beside the copy peak of MEASURED_PEAKS.json."""
    import ctypes

    import torch
    try:
        lib = ctypes.CDLL(build_readbw())
    except Exception:
        return None, "unavailable (tools/readbw.cu did not build)"
    lib.readbw.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_void_p]
    flat = gb.pool.view(-1)
    nbytes = min(4 << 30, flat.numel() * flat.element_size()) // 16 * 16
    source = "the KV pool"
    if nbytes < (1 << 30):       # a small pool (c1: 8 MB) would measure latency, not bandwidth
        flat = torch.ones(1 << 30, dtype=torch.int32, device="cuda")
        nbytes = flat.numel() * flat.element_size()
        source = "a 4 GiB scratch buffer (the KV pool is < 1 GiB)"
    sink = torch.zeros(4096, dtype=torch.int32, device="cuda")
    best = 0.0
    for rep in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.readbw(flat.data_ptr(), nbytes, sink.data_ptr(), 1184, 512, 8, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if rep >= 2:
            best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return (round(best, 1), source) if best > 0 else (None, source)


# --------------------------------------------------------------------- neo arm


def run_neo(args):
    import torch
    import torch.distributed as dist

    from neo_inputs.gpu import GpuBatch
    from neo_inputs.workloads import WORKLOADS
    from paper_2411_01142_b200 import neo

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and rank == 0:
        print(f"note: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    # Harness check on ONE GPU (never a measurement): NEO_BENCH_DIST_BACKEND=gloo
    # with NEO_BENCH_SHARE_GPU=1 runs every rank on cuda:0 with gloo collectives
    # on host copies, so the multi-rank code paths (rank plans, per-rank timing,
    # aggregation, head reassembly) execute end to end under torchrun.
    global COLL_DEV
    backend = os.environ.get("NEO_BENCH_DIST_BACKEND", "nccl")
    COLL_DEV = "cpu" if backend == "gloo" else "cuda"
    if os.environ.get("NEO_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.config]
    ctx_all, req_ids, kvh, qh, scaling, par = shard_plan(wl, rank, world, args.fraction)
    # harness only (with NEO_BENCH_SHARE_GPU=1): fewer distinct layer pools, cycled,
    # so several full-size ranks fit on one GPU; never set for a measurement
    max_pools = os.environ.get("NEO_BENCH_MAX_POOLS") if os.environ.get("NEO_BENCH_SHARE_GPU") == "1" else None
    gb = GpuBatch(wl, ctx=ctx_all, req_ids=req_ids, kv_heads=kvh, q_heads=qh,
                  layers=min(wl.layers_built, int(max_pools)) if max_pools else None)
    L = layers_per_step(wl)
    stream = torch.cuda.current_stream()
    # a0 plan from the host-known lengths (NEO's scheduler holds them)
    chunk = args.chunk or neo.plan_chunk(gb.ctx, gb.hkv, gb.P)
    ws = neo.make_workspace(gb.B, gb.hq, gb.hkv, gb.max_seq_len, chunk)
    out = torch.empty(L, gb.B, gb.hq, 128, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()

    # every layer call reads KV that no kernel of the step writes (one
    # attention launch per layer over immutable earlier-token pages), so the
    # calls declare NEO_ATTN_KV_STABLE (include/neo.h)
    kv_stable = not args.no_kv_stable

    def attn_layer(l):
        k, v = gb.layer(l)
        neo.decode_attn(gb.q[l % gb.layers], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=out[l],
                        chunk_tokens=chunk, workspace=ws, stream=stream, kv_stable=kv_stable)

    def step(events=None):
        for l in range(L):
            attn_layer(l)
            if events is not None:
                events[l].record(stream)

    graph = None
    if args.graph:
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()

    # Small configs (c1: 8 MB of KV) would be served from the 126 MB L2 across
    # steps: flush it by READING a 512 MB buffer before every step (clean lines,
    # so no write-backs compete with the timed kernel), outside the timed
    # attention window.  Big configs cycle >= 4 GB of distinct KV per step.
    flush = None
    if gb.layers * gb.kv_bytes_per_call() < 1e9:
        flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")

    for _ in range(args.warmup):
        if flush is not None:
            flush.sum()
        step() if graph is None else graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    # Timed region: events only at step boundaries, so consecutive launches stay
    # back to back (and programmatic dependent launch can overlap them).
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for s in range(args.steps):
        if flush is not None:
            flush.sum()
        starts[s].record(stream)
        step() if graph is None else graph.replay()
        ends[s].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [starts[s].elapsed_time(ends[s]) for s in range(args.steps)]
    t_ms = sum(step_ms)
    # Per-launch durations of the attention kernel for the roofline: a separate
    # pass with an event after every launch, on the launching stream.
    launch_ms = []
    for s in range(min(args.steps, 3)):
        per = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
        st = torch.cuda.Event(enable_timing=True)
        if flush is not None:
            flush.sum()
        st.record(stream)
        step(per)
        torch.cuda.synchronize()
        prev = st
        for l in range(L):
            launch_ms.append(prev.elapsed_time(per[l]))
            prev = per[l]
    kv_local = gb.kv_bytes_per_call() * L * args.steps
    tok_local = int(gb.ctx.astype(np.int64).sum()) * L * args.steps
    t_max, kv_total, tok_total, per_rank = aggregate_ranks(t_ms / 1e3, kv_local, tok_local, args.steps, world,
                                                           head_sharded=(wl.name == "c4"), dist=dist,
                                                           device=COLL_DEV)
    value = kv_total / t_max / 1e9
    # The step is exactly L back-to-back launches of the decode kernel and nothing
    # else on the stream (profiles/r02_launches_c3.md: 100 % of the timed
    # kernels), so its average launch duration is the rank's step time / L --
    # timed with programmatic dependent launch intact.  The event-per-launch pass
    # above breaks that overlap; it is reported only as `isolated_launch_us`.
    avg_launch = t_ms / 1e3 / (L * args.steps)
    hbm_peak, peak_src = peaks()
    read_ceiling, rc_source = measure_read_ceiling(gb, stream)
    algo = gb.kv_bytes_per_call() + gb.other_bytes_per_call()
    achieved = algo / avg_launch / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if world == 1 and os.path.exists(tpath):       # the committed ncu captures are 1-GPU launches
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, gb, L, chunk, ws, stream, world, dist)

    reassembly = None
    if wl.name == "c4" and world > 1:
        reassembly = run_reassembly(args, gb, L, step, stream, world, dist)

    cpu_share = None
    if wl.name == "c5" and args.fraction < 1.0 and rank == 0:
        cpu_share = run_cpu_share(args, wl, ctx_all, int(round(args.fraction * len(ctx_all))), t_max / (L * args.steps))

    swap = None
    if wl.swap_requests and not args.no_swap:
        swap = run_swap(args, gb, L, step, attn_layer, stream)

    prefill = None
    if rank == 0 and not args.no_prefill:
        prefill = run_prefill(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(gb, target_s=10.0)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_max * 1e3 / args.steps, 4),
            "ms_per_step_rank0": {"median": round(float(np.median(step_ms)), 4), "min": round(min(step_ms), 4),
                                  "max": round(max(step_ms), 4)},
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (counter-based generator, LLaMa shapes; no weights needed)",
            "attended_tokens_per_s": round(tok_total / t_max, 1),
            "pct_of_measured_hbm": round(100 * value / world / hbm_peak, 2),
            "pct_of_nominal_hbm": round(100 * value / world / NOMINAL_HBM_GBS, 2),
            "config": {
                "workload": f"{wl.name}: {wl.model} {wl.note}",
                "batch": batch_total(wl, gb, world, args.fraction, ctx_all),
                "batch_per_rank": gb.B,
                "q_heads": wl.hq, "kv_heads": wl.hkv, "head_dim": 128, "page_size": wl.page_size,
                "seq_len_mean": round(float(gb.ctx.mean()), 1), "seq_len_min": int(gb.ctx.min()),
                "seq_len_max": int(gb.ctx.max()),
                "layers_per_step": L, "distinct_layer_pools": gb.layers,
                "chunk_tokens": chunk, "chunk_mode": f"grouped (groups <= {4096 // -chunk if chunk >= -4 else -chunk} tokens)" if chunk < 0
                else "split",
                "chunk_plan": "explicit --chunk" if args.chunk else
                "neo_decode_attn_plan_chunk (host lengths)", "parallelism": par,
                "l2": (f"inputs {gb.layers * gb.kv_bytes_per_call() / 1e9:.1f} GB of distinct KV cycled per step "
                       ">> 126 MB L2; no flush") if flush is None else
                      "L2 flushed (512 MB read) before every step, outside the timed attention window",
                "cuda_graph": bool(graph is not None),
                "kv_stable": kv_stable,
            },
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                         "kernel": "decode_attn_group_kernel" if chunk < 0 else
                         "decode_attn_kernel", "avg_launch_us": round(avg_launch * 1e6, 2),
                         "avg_launch_source": "rank-0 timed step / launches per step (PDL intact)",
                         "isolated_launch_us": round(float(np.mean(launch_ms)) * 1e3, 2),
                         "algorithmic_bytes_per_launch": algo, "peak_source": peak_src,
                         "read_ceiling_gbs": read_ceiling,
                         "frac_of_read_ceiling": round(achieved / read_ceiling, 4) if read_ceiling else None,
                         "frac_of_nominal": round(achieved / NOMINAL_HBM_GBS, 4),
                         "read_ceiling_source": "measured in this run: 16-byte non-allocating loads over up to 4 GiB "
                                                f"of {rc_source}, 1184 CTAs x 512 threads, best of 5 (tools/readbw.cu)"},
            "per_rank_ms_per_step": None if per_rank is None else [round(x, 4) for x in per_rank],
            "rank_imbalance": None if per_rank is None else rank_imbalance(per_rank),
            "gpu_launches": L * args.steps,
            "clocks": clk,
            "e2e": e2e,
            "swap": swap,
            "reassembly": reassembly,
            "cpu_share": cpu_share,
            "prefill": prefill,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def tensor_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3, burst)"
    except Exception:
        return 2250.0, "nominal dense bf16 2.25 PFLOP/s (no measured peak)"


def run_prefill(args):
    """the prefill half of NEO's batch-0 for one
    LLaMa-3.1-8B layer -- whole prompts of ~1000 tokens (P:364's synthetic
    input length, lengths uniform in [0.9 l, 1.1 l]) up to max_batch_tokens 8192:
    neo_prefill_append (K/V store + RoPE) then neo_prefill_attn, each timed per
    launch with CUDA events on the launching stream, L2 flushed between reps."""
    import torch

    from paper_2411_01142_b200 import neo
    hq, hkv, d, P = 32, 8, 128, 16
    rng = np.random.default_rng(0x4E454F)
    lens = []
    while True:
        n = int(rng.integers(900, 1101))
        if sum(lens) + n > 8192:
            break
        lens.append(n)
    B, T = len(lens), sum(lens)
    npg = [(n + P - 1) // P for n in lens]
    g = torch.Generator(device="cuda").manual_seed(7)
    k_pages = torch.randn(sum(npg) + 4, hkv, P, d, device="cuda", dtype=torch.bfloat16, generator=g)
    v_pages = torch.randn(sum(npg) + 4, hkv, P, d, device="cuda", dtype=torch.bfloat16, generator=g)
    perm = torch.randperm(sum(npg), device="cuda", generator=g).to(torch.int32)
    bt = torch.zeros(B, max(npg), dtype=torch.int32, device="cuda")
    o = 0
    for b, m in enumerate(npg):
        bt[b, :m] = perm[o:o + m]
        o += m
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    qo = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    q = torch.randn(T, hq, d, device="cuda", dtype=torch.bfloat16, generator=g)
    kn = torch.randn(T, hkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
    vn = torch.randn(T, hkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
    inv = (500000.0 ** (-torch.arange(0, d, 2, dtype=torch.float64) / d)).float().cuda()
    out = torch.empty_like(q)
    flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    app, att = [], []
    for rep in range(3 + 10):
        flush.sum()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        neo.prefill_append(k_pages, v_pages, bt, sl, qo, kn, vn, q=q, inv_freq=inv)
        e[1].record(stream)
        neo.prefill_attn(q, k_pages, v_pages, bt, sl, qo, max(lens), out=out)
        e[2].record(stream)
        torch.cuda.synchronize()
        if rep >= 3:
            app.append(e[0].elapsed_time(e[1]) / 1e3)
            att.append(e[1].elapsed_time(e[2]) / 1e3)
    flops = sum(4.0 * d * hq * n * (n + 1) / 2 for n in lens)
    t_att = float(np.mean(att))
    long_prompt = run_prefill_long(flush)
    # the launch picks the stream kernel for prompts up to 3072 tokens (neo_prefill.cu kStreamMaxQLen)
    kernel = "prefill_attn_stream_kernel" if max(lens) <= 3072 else "prefill_attn_kernel"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):          # ncu --set full of this launch (profiles/r02_ncu_full_prefill_stream.md)
        traffic = json.load(open(tpath)).get("prefill_stream" if kernel.endswith("stream_kernel") else "prefill")
    peak, src = tensor_peak()
    achieved = flops / t_att / 1e12
    return {
        "workload": f"LLaMa-3.1-8B layer (32/8 heads, D 128, P 16): {B} whole prompts, {T} tokens "
                    f"(lengths U[900, 1100] up to max_batch_tokens 8192)",
        "data": "synthetic N(0,1) bf16, seeded",
        "attn_us": round(t_att * 1e6, 2), "append_rope_us": round(float(np.mean(app)) * 1e6, 2),
        "gpu_launches": 2 * 10,
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kernel,
                     "algorithmic_flops_per_launch": flops, "peak_source": src,
                     "algorithmic_bytes_per_launch": T * (2 * hq + 2 * hkv) * d * 2,
                     "mma_flops_per_algorithmic_flop": 1.0,
                     "note": "algorithmic = causal 4*D per (q-head, row, visible key); prompts >= 256 tokens run "
                             "P.V in fp16 (one MMA per K16 step, DESIGN reading n1), so the tensor core executes "
                             "these flops (plus the masked halves of diagonal tiles)"},
        "l2": "flushed (512 MB read) before every rep",
        "long_prompt": long_prompt,
    }


def run_prefill_long(flush, n=16384):
    """The same kernel on one whole 16K-token prompt (the long end of P:364's
    mixes; the steady state without item switches), for context beside the
    NEO-sized leg above."""
    import torch

    from paper_2411_01142_b200 import neo
    hq, hkv, d, P = 32, 8, 128, 16
    g = torch.Generator(device="cuda").manual_seed(11)
    npg = n // P
    k_pages = torch.randn(npg, hkv, P, d, device="cuda", dtype=torch.bfloat16, generator=g)
    v_pages = torch.randn(npg, hkv, P, d, device="cuda", dtype=torch.bfloat16, generator=g)
    bt = torch.randperm(npg, device="cuda", generator=g).to(torch.int32).view(1, npg)
    sl = torch.tensor([n], dtype=torch.int32, device="cuda")
    qo = torch.tensor([0, n], dtype=torch.int32, device="cuda")
    q = torch.randn(n, hq, d, device="cuda", dtype=torch.bfloat16, generator=g)
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    ts = []
    for rep in range(2 + 5):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        neo.prefill_attn(q, k_pages, v_pages, bt, sl, qo, n, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.mean(ts))
    flops = 4.0 * d * hq * n * (n + 1) / 2
    peak, src = tensor_peak()
    return {"workload": f"1 whole prompt of {n} tokens, LLaMa-3.1-8B layer shapes", "attn_us": round(t * 1e6, 1),
            "achieved_tflops": round(flops / t / 1e12, 1), "frac": round(flops / t / 1e12 / peak, 4),
            "peak": peak}


def run_cpu_share(args, wl, ctx_all, n_gpu, t_ga):
    """NEXT-2 in NEO's asymmetric setting (c5, f < 1): the CPU-resident requests
    [n_gpu, 1024) are swapped out to the pinned CPU-cache with the product's own
    neo_kv_swap_out, then their decode attention runs on the host cores with
    neo_cpu_decode_attn (T_ca), next to the GPU's per-layer time T_ga.
    Also times the per-layer TrQKV / TrO transfers of those requests."""
    import torch

    from neo_inputs.gpu import GpuBatch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo
    ids = np.arange(n_gpu, len(ctx_all))
    if len(ids) == 0:
        return None
    cb = GpuBatch(wl, ctx=ctx_all, req_ids=ids, layers=1)
    pool = neo.KVPool(1, cb.hkv, cb.num_pages, num_host_pages=cb.num_pages, page_size=cb.P, gpu_buffer=cb.pool)
    gids = pool.alloc(NEO_GPU, cb.num_pages)
    hids = pool.alloc(NEO_HOST, cb.num_pages)
    assert np.array_equal(gids, np.arange(cb.num_pages)) and np.array_equal(hids, np.arange(cb.num_pages))
    staging = torch.empty(min(pool.staging_bytes(cb.num_pages), 1 << 30), dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pool.swap_out(gids, hids, staging)                     # host page id == GPU page id
    e1.record()
    torch.cuda.synchronize()
    swap_ms = e0.elapsed_time(e1)
    q_host = cb.q[0].cpu()
    nth = ncores()
    out = pool.cpu_decode_attn(0, q_host, cb.table, cb.ctx, num_threads=nth)   # warm-up
    reps, t = 0, 0.0
    while reps < 3 or (t < 5.0 and reps < 50):
        t0 = time.time()
        pool.cpu_decode_attn(0, q_host, cb.table, cb.ctx, out=out, num_threads=nth)
        t += time.time() - t0
        reps += 1
    t_ca = t / reps
    kvb = cb.kv_bytes_per_call()
    # TrQKV (q, k, v of the new token of every CPU-request, device -> host) and
    # TrO (attention output, host -> device), per layer, pinned memory
    nq = len(ids) * wl.hq * 128 * 2
    nkv = len(ids) * wl.hkv * 128 * 2 * 2
    dev = torch.empty(nq + nkv, dtype=torch.uint8, device="cuda")
    hst = torch.empty(nq + nkv, dtype=torch.uint8).pin_memory()
    e0.record()
    hst.copy_(dev, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    tr_qkv = e0.elapsed_time(e1)
    e0.record()
    dev[:nq].copy_(hst[:nq], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    tr_o = e0.elapsed_time(e1)
    res = {"requests": int(len(ids)), "kv_bytes": int(kvb), "threads": nth, "cpu": cpu_model(),
           "t_ca_ms": round(t_ca * 1e3, 3), "cpu_attention_gbs": round(kvb / t_ca / 1e9, 3),
           "t_ga_ms_gpu_share": round(t_ga * 1e3, 4), "swap_out_ms": round(swap_ms, 3),
           "trqkv_bytes": int(nq + nkv), "trqkv_ms": round(tr_qkv, 4), "tro_bytes": int(nq), "tro_ms": round(tr_o, 4)}
    pool.close()
    del cb
    torch.cuda.empty_cache()
    return res


def run_reassembly(args, gb, L, step, stream, world, dist):
    """a9 (multi-GPU, head-sharded c4): after each layer's attention, reassemble
    the full-head output with one all_gather_into_tensor over NVLink (NCCL) on a
    communication stream, overlapped with the next layer's attention (SURVEY
    §8(e)).  Reported separately from the attention-only value."""
    import torch

    from paper_2411_01142_b200 import neo
    comm = torch.cuda.Stream()
    full = torch.empty((L, gb.B, gb.hq * world, 128), dtype=torch.bfloat16, device="cuda")
    gbuf = torch.empty((L, world, gb.B, gb.hq, 128), dtype=torch.bfloat16, device="cuda")
    outl = torch.empty((L, gb.B, gb.hq, 128), dtype=torch.bfloat16, device="cuda")
    chunk = neo.plan_chunk(gb.ctx, gb.hkv, gb.P)
    ws = neo.make_workspace(gb.B, gb.hq, gb.hkv, gb.max_seq_len, chunk)
    evs = [torch.cuda.Event() for _ in range(L)]

    def step_gather():
        for l in range(L):
            k, v = gb.layer(l)
            neo.decode_attn(gb.q[l % gb.layers], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, out=outl[l],
                            chunk_tokens=chunk, workspace=ws, stream=stream)
            evs[l].record(stream)
            comm.wait_event(evs[l])
            with torch.cuda.stream(comm):
                if COLL_DEV == "cpu":      # gloo harness check: host copies
                    hb = torch.empty(gbuf[l].numel() // 2, dtype=torch.int32)     # (gloo has no 16-bit types)
                    dist.all_gather_into_tensor(hb, outl[l].view(-1).view(torch.int32).cpu())
                    gbuf[l].view(-1).view(torch.int32).copy_(hb)
                else:
                    dist.all_gather_into_tensor(gbuf[l].view(-1), outl[l].view(-1))
                reassemble_heads_into(full[l], gbuf[l])
        stream.wait_stream(comm)

    for _ in range(2):
        step_gather()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step_gather()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=COLL_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"ms_per_step_with_allgather": round(float(t.item()), 4),
            "allgather_bytes_per_layer_per_rank": int(outl[0].numel() * 2),
            "overlap": "all_gather of layer l on a comm stream while layer l+1 computes"}


def run_swap(args, gb, L, step, attn_layer, stream):
    """c3's a8 row: swap the last `swap_requests` requests (LIFO victims)
    out to pinned host through neo_kv_swap_out on a side stream (gather kernel +
    cudaMemcpy2DAsync over PCIe), alone and concurrently with attention steps;
    compare with a plain pinned D2H memcpy of the same bytes; swap back in."""
    import torch

    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo
    wl = gb.wl
    victims = np.arange(gb.B - wl.swap_requests, gb.B)
    need = (gb.ctx + gb.P - 1) // gb.P
    gpu_ids = np.concatenate([gb.table[b, :need[b]] for b in victims]).astype(np.int32)
    n = len(gpu_ids)
    pool = neo.KVPool(gb.layers, gb.hkv, gb.num_pages, num_host_pages=n, page_size=gb.P, gpu_buffer=gb.pool)
    pool.alloc(NEO_GPU, gb.num_pages)                # every page of the batch is in use
    host_ids = pool.alloc(NEO_HOST, n)
    nbytes = pool.staging_bytes(n)
    staging = torch.empty(min(nbytes, 1 << 30), dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    torch.cuda.synchronize()

    def timed(fn, s):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        return e0, e1

    pool.swap_out(gpu_ids[:8], host_ids[:8], staging, stream=side)        # warm-up
    torch.cuda.synchronize()
    a, b = timed(lambda: pool.swap_out(gpu_ids, host_ids, staging, stream=side), side)
    torch.cuda.synchronize()
    t_out = a.elapsed_time(b) / 1e3
    # plain pinned D2H memcpy of the same number of bytes (PCIe ceiling for this path)
    dev = gb.pool.view(-1)[: nbytes // 2]
    hostv = pool.host.view(-1)[: nbytes // 2]
    def d2h():
        with torch.cuda.stream(side):
            hostv.copy_(dev, non_blocking=True)

    def h2d():
        with torch.cuda.stream(side):
            dev.copy_(hostv, non_blocking=True)

    a, b = timed(d2h, side)
    torch.cuda.synchronize()
    t_d2h = a.elapsed_time(b) / 1e3
    # swap-in back to the same pages (H2D + scatter)
    a, b = timed(lambda: pool.swap_in(host_ids, gpu_ids, staging, stream=side), side)
    torch.cuda.synchronize()
    t_in = a.elapsed_time(b) / 1e3
    a, b = timed(h2d, side)
    torch.cuda.synchronize()
    t_h2d = a.elapsed_time(b) / 1e3
    # zero-copy variant: the kernel stores straight into the mapped pinned pages
    a, b = timed(lambda: pool.swap_out(gpu_ids, host_ids, None, stream=side), side)
    torch.cuda.synchronize()
    t_zc_out = a.elapsed_time(b) / 1e3
    a, b = timed(lambda: pool.swap_in(host_ids, gpu_ids, None, stream=side), side)
    torch.cuda.synchronize()
    t_zc_in = a.elapsed_time(b) / 1e3
    # attention while a swap-out runs on the side stream
    steps = max(2, min(args.steps, 5))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    sa, sb = timed(lambda: pool.swap_out(gpu_ids, host_ids, staging, stream=side), side)
    enqueue_ms = (time.perf_counter() - h0) * 1e3
    s0.record(stream)
    for _ in range(steps):
        step()
    s1.record(stream)
    torch.cuda.synchronize()
    t_att = s0.elapsed_time(s1) / 1e3
    pool.swap_in(host_ids, gpu_ids, staging, stream=side)              # restore
    torch.cuda.synchronize()
    # NEXT-1 layer-wise pipeline ("start PCIe transmission immediately
    # after each layer's KV value is computed"): in one decode step, right after
    # layer l's attention the victims' layer-l pages go out on the side stream
    # (neo_kv_swap_out_ex + NEO_SWAP_DEFER_JOIN, so the library overlaps layer
    # l+1's gather with layer l's D2H through the two staging halves); one
    # neo_kv_swap_join ends the step's swap.
    def layerwise():
        ev = [torch.cuda.Event() for _ in range(L)]
        e_st, e_att = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_sw0, e_sw1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_st.record(stream)
        for l in range(L):
            attn_layer(l)
            ev[l].record(stream)
            side.wait_event(ev[l])
            if l == 0:
                e_sw0.record(side)
            pool.swap_out(gpu_ids, host_ids, staging, l % gb.layers, l % gb.layers + 1, stream=side,
                          defer_join=True)
        e_att.record(stream)
        pool.swap_join(stream=side)
        e_sw1.record(side)
        torch.cuda.synchronize()
        return e_st.elapsed_time(e_att) / 1e3, e_sw0.elapsed_time(e_sw1) / 1e3, e_st.elapsed_time(e_sw1) / 1e3

    layerwise()                                                        # warm-up
    lw = [layerwise() for _ in range(2)]
    lw_att, lw_swap, lw_total = (float(np.mean([x[i] for x in lw])) for i in range(3))
    lw_bytes = nbytes * L // gb.layers
    pool.close()
    return {"requests": int(wl.swap_requests), "pages": int(n), "layers": int(gb.layers), "bytes": int(nbytes),
            "swap_out_gbs": round(nbytes / t_out / 1e9, 2), "swap_in_gbs": round(nbytes / t_in / 1e9, 2),
            "pcie_d2h_memcpy_gbs": round(nbytes / t_d2h / 1e9, 2),
            "pcie_h2d_memcpy_gbs": round(nbytes / t_h2d / 1e9, 2),
            "swap_out_frac_of_memcpy": round(t_d2h / t_out, 4),
            "zero_copy_swap_out_gbs": round(nbytes / t_zc_out / 1e9, 2),
            "zero_copy_swap_in_gbs": round(nbytes / t_zc_in / 1e9, 2),
            "attention_gbs_during_swap": round(gb.kv_bytes_per_call() * L * steps / t_att / 1e9, 2),
            "attention_steps_during_swap": steps, "staging_bytes": int(staging.numel()),
            "swap_outlasted_attention": bool(sa.elapsed_time(s1) < sa.elapsed_time(sb)),
            "concurrent_leg": {"swap_enqueue_host_ms": round(enqueue_ms, 3),
                               "attention_start_after_swap_start_ms": round(sa.elapsed_time(s0), 3),
                               "attention_end_after_swap_start_ms": round(sa.elapsed_time(s1), 3),
                               "swap_ms": round(sa.elapsed_time(sb), 3)},
            "layerwise_pipeline": {
                "what": "per decode step: attention(l) on the main stream, then swap-out of the 16 victims' "
                        "layer-l pages on a side stream (neo_kv_swap_out_ex, NEO_SWAP_DEFER_JOIN; staging split "
                        "in two halves by the library), one neo_kv_swap_join per step",
                "bytes": int(lw_bytes), "calls_per_step": int(L),
                "attention_gbs": round(gb.kv_bytes_per_call() * L / lw_att / 1e9, 2),
                "swap_gbs": round(lw_bytes / lw_swap / 1e9, 2),
                "swap_frac_of_memcpy": round((lw_bytes / lw_swap) / (nbytes / t_d2h), 4),
                "step_ms_incl_swap": round(lw_total * 1e3, 3), "attention_ms": round(lw_att * 1e3, 3),
                "swap_ms_from_first_layer": round(lw_swap * 1e3, 3)}}


def run_e2e(args, gb, L, chunk, ws, stream, world, dist):
    """The same metric end to end through the public API: every step copies its
    inputs (q of every layer, block table, seq_lens) host->device from pinned
    memory, runs the L attention calls and copies every layer's output back to
    pinned host memory.  Copies run on two copy streams, pipelined per layer with
    the attention launches, into two device buffer sets used by alternate steps
    (the next step's uploads and this step's downloads overlap compute); the
    timed region ends when the last step's outputs have reached the host."""
    import torch

    from paper_2411_01142_b200 import neo
    q_host = torch.empty((L, gb.B, gb.hq, 128), dtype=torch.bfloat16).pin_memory()
    for l in range(L):
        q_host[l].copy_(gb.q[l % gb.layers])
    bt_host = gb.block_table.cpu().pin_memory()
    sl_host = gb.seq_lens.cpu().pin_memory()
    out_host = torch.empty((L, gb.B, gb.hq, 128), dtype=torch.bfloat16).pin_memory()
    # two device buffer sets, alternating by step: step s+1 uploads while step s
    # computes, and step s's outputs download while step s+1 computes
    q_dev = [torch.empty_like(q_host, device="cuda") for _ in range(2)]
    bt_dev = [torch.empty_like(bt_host, device="cuda") for _ in range(2)]
    sl_dev = [torch.empty_like(sl_host, device="cuda") for _ in range(2)]
    out_dev = [torch.empty_like(out_host, device="cuda") for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [[torch.cuda.Event() for _ in range(L)] for _ in range(2)]
    ev_att = [[torch.cuda.Event() for _ in range(L)] for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]      # compute finished reading set i
    ev_down = [torch.cuda.Event() for _ in range(2)]      # outputs of set i reached the host
    for i in range(2):
        ev_used[i].record(stream)
        ev_down[i].record(stream)
    counter = [0]

    def step():
        i = counter[0] % 2
        counter[0] += 1
        h2d_s.wait_event(ev_used[i])               # the step two back finished with set i
        with torch.cuda.stream(h2d_s):
            bt_dev[i].copy_(bt_host, non_blocking=True)
            sl_dev[i].copy_(sl_host, non_blocking=True)
            for l in range(L):
                q_dev[i][l].copy_(q_host[l], non_blocking=True)
                ev_in[i][l].record(h2d_s)
        stream.wait_event(ev_down[i])              # its outputs were downloaded before overwriting
        for l in range(L):
            stream.wait_event(ev_in[i][l])
            k, v = gb.layer(l)
            neo.decode_attn(q_dev[i][l], k, v, bt_dev[i], sl_dev[i], gb.max_seq_len, out=out_dev[i][l],
                            chunk_tokens=chunk, workspace=ws, stream=stream, kv_stable=not args.no_kv_stable)
            ev_att[i][l].record(stream)
        ev_used[i].record(stream)
        with torch.cuda.stream(d2h_s):
            for l in range(L):
                d2h_s.wait_event(ev_att[i][l])
                out_host[l].copy_(out_dev[i][l], non_blocking=True)
            ev_down[i].record(d2h_s)

    def drain():
        for i in range(2):
            stream.wait_event(ev_down[i])

    for _ in range(max(1, args.warmup)):
        step()
    drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    drain()                                        # every step's outputs are on the host
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=COLL_DEV)
    kv = torch.tensor([float(gb.kv_bytes_per_call() * L * args.steps)], dtype=torch.float64, device=COLL_DEV)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(kv, op=dist.ReduceOp.SUM)
    h2d = q_host.numel() * 2 + bt_host.numel() * 4 + sl_host.numel() * 4
    return {"value": round(float(kv.item()) / float(t.item()) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(out_host.numel() * 2),
            "ms_per_step": round(float(t.item()) * 1e3 / args.steps, 4)}


# ------------------------------------------------------------- CPU oracle legs


def ncores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample_inputs(wl, ctx, req_ids, layer, heads=None, qheads=None):
    import neo_inputs as ni
    qs, ks, vs = [], [], []
    kvh = np.arange(*(heads or (0, wl.hkv)))
    qh = np.arange(*(qheads or (0, wl.hq)))
    for b in req_ids:
        n = int(ctx[b])
        qs.append(ni.q_bits(wl.seed, layer, [int(b)], wl.hq, 128, heads=qh)[0])
        ks.append(ni.kv_bits(wl.seed, layer, ni.KIND_K, int(b), 0, n, wl.hkv, 128, heads=kvh))
        vs.append(ni.kv_bits(wl.seed, layer, ni.KIND_V, int(b), 0, n, wl.hkv, 128, heads=kvh))
    return np.stack(qs), ks, vs


def cpu_baseline(gb, target_s=10.0):
    """The fp64 oracle (as it stands) on this box's host cores over a bounded
    sample of the same workload: requests of layer 0, threads over requests."""
    import oracle
    wl = gb.wl
    ids_local = np.arange(gb.B)
    gids = gb.req_ids
    nth = ncores()
    ctx_g = np.zeros(int(gids.max()) + 1, dtype=np.int64)
    ctx_g[gids] = gb.ctx
    # calibrate on a few requests, then size the sample for ~target_s
    cal = gids[:max(1, min(len(gids), nth))]
    q, k, v = oracle_sample_inputs(wl, ctx_g, cal, 0, gb.kv_heads, gb.q_heads)
    t0 = time.time()
    oracle.decode_attention_batch(q, k, v, 1 / math.sqrt(128), nthreads=nth)
    dt = max(time.time() - t0, 1e-3)
    tok_per_s = float(ctx_g[cal].sum()) / dt
    want_tokens = tok_per_s * target_s
    cum = np.cumsum(gb.ctx)
    n = int(min(len(ids_local), max(len(cal), np.searchsorted(cum, want_tokens) + 1)))
    sample = gids[:n]
    q, k, v = oracle_sample_inputs(wl, ctx_g, sample, 0, gb.kv_heads, gb.q_heads)
    # repeat the sample until ~target_s of CPU work has been timed
    reps, dt = 0, 0.0
    while dt < target_s and reps < 1000:
        t0 = time.time()
        oracle.decode_attention_batch(q, k, v, 1 / math.sqrt(128), nthreads=nth)
        dt += time.time() - t0
        reps += 1
    toks = int(ctx_g[sample].sum()) * reps
    kvb = toks * gb.hkv * 128 * 2 * 2
    return {"value": round(kvb / dt / 1e9, 4), "unit": "GB/s", "cores": nth, "kind": "oracle",
            "sample": f"{n} of {gb.B} requests of layer 0 ({int(ctx_g[sample].sum())} tokens, "
                      f"{kvb / reps / 1e9:.2f} GB of KV) x {reps} repetitions, fp64 C oracle, pthreads over "
                      f"requests; {cpu_model()}",
            "attended_tokens_per_s": round(toks / dt, 1), "seconds": round(dt, 2)}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle, timed on the host cores, on the same
    config/metric; each step a bounded sample of the workload (layer = step % L)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    import oracle
    from neo_inputs.workloads import WORKLOADS
    wl = WORKLOADS[args.config]
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    ctx_all, req_ids, kvh, qh, scaling, par = shard_plan(wl, 0, 1, args.fraction)
    ids = np.arange(len(ctx_all)) if req_ids is None else req_ids
    nth = ncores()
    total_budget = 150.0
    per_step = max(0.5, total_budget / max(1, args.steps + args.warmup))
    cal = ids[:max(1, min(len(ids), nth))]
    q, k, v = oracle_sample_inputs(wl, ctx_all, cal, 0, kvh, qh)
    t0 = time.time()
    oracle.decode_attention_batch(q, k, v, 1 / math.sqrt(128), nthreads=nth)
    tok_rate = float(ctx_all[cal].sum()) / max(time.time() - t0, 1e-3)
    cum = np.cumsum(ctx_all[ids])
    n = int(min(len(ids), max(len(cal), np.searchsorted(cum, tok_rate * per_step) + 1)))
    sample = ids[:n]
    hkv = wl.hkv if kvh is None else kvh[1] - kvh[0]
    L = layers_per_step(wl)
    inputs = [oracle_sample_inputs(wl, ctx_all, sample, l, kvh, qh) for l in range(min(L, 2))]
    for s in range(args.warmup):
        q, k, v = inputs[s % len(inputs)]
        oracle.decode_attention_batch(q, k, v, 1 / math.sqrt(128), nthreads=nth)
    t0 = time.time()
    for s in range(args.steps):
        q, k, v = inputs[s % len(inputs)]
        oracle.decode_attention_batch(q, k, v, 1 / math.sqrt(128), nthreads=nth)
    dt = time.time() - t0
    toks = int(ctx_all[sample].sum()) * args.steps
    kvb = toks * hkv * 128 * 2 * 2
    value = kvb / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 3),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator and workload as the neo arm)",
        "attended_tokens_per_s": round(toks / dt, 1),
        "config": {"workload": f"{wl.name}: {wl.model} {wl.note}", "parallelism": "host cores (no GPU)",
                   "sample_requests": int(n), "batch": int(len(ids))},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": nth, "kind": "oracle",
                         "sample": f"{n} of {len(ids)} requests per step (one layer), fp64 C oracle, {cpu_model()}"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_neo(args)


if __name__ == "__main__":
    main()
