"""Partitioning of the decode-attention work across B200s.

* By KV head (tensor parallel: "each responsible for a portion of
  KV heads"): rank r owns kv heads [r*Hkv/N, (r+1)*Hkv/N) and the q heads
  [r*Hq/N, (r+1)*Hq/N) that attend to them (contiguous because g = floor(h/G)).
  No collective inside attention; outputs are reassembled with an all-gather only
  where a consumer needs full heads.
* By request (data parallel): longest-processing-time-first greedy on seq_len,
  ties by request id, deterministic.  No collective on the data path.
"""
from __future__ import annotations

import numpy as np


def head_shard(hq: int, hkv: int, rank: int, world: int):
    """((kv_begin, kv_end), (q_begin, q_end)) owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if hkv % world:
        raise ValueError("world size must divide num_kv_heads")
    per = hkv // world
    G = hq // hkv
    return (rank * per, (rank + 1) * per), (rank * per * G, (rank + 1) * per * G)


def lpt_assign(ctx, world: int) -> list[np.ndarray]:
    """Request ids of each rank (sorted), LPT on seq_len, ties by id."""
    ctx = np.asarray(ctx)
    order = sorted(range(len(ctx)), key=lambda i: (-int(ctx[i]), i))
    load = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(ctx[i])
    return [np.array(sorted(x), dtype=np.int64) for x in out]


def gather_heads(local_out, world: int, group=None):
    """Reassemble head-sharded outputs [B][Hq/N][D] -> [B][Hq][D] with one
    all_gather_into_tensor (NCCL over NVLink on GPUs, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist
    B, hl, D = local_out.shape
    buf = torch.empty((world, B, hl, D), dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(buf.view(-1), local_out.contiguous().view(-1), group=group)
    return buf.permute(1, 0, 2, 3).reshape(B, world * hl, D)
