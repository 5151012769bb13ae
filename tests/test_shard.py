"""Multi-GPU partitioning logic on CPU: head sharding (TP,
P:312-314) and LPT request sharding cover every unit exactly once, and the
world-size-2 gloo path (shard -> per-rank attention -> all_gather) reassembles
exactly the single-process result.  Per-rank attention here is the oracle
(CPU); the CUDA kernel's per-shard parity is tests/test_gpu_fullsize.py."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_01142_b200.shard import gather_heads, head_shard, lpt_assign


@pytest.mark.parametrize("hq,hkv,world", [(64, 8, 1), (64, 8, 2), (64, 8, 4), (64, 8, 8), (32, 8, 4)])
def test_head_shard_partition(hq, hkv, world):
    kv_seen, q_seen = [], []
    G = hq // hkv
    for r in range(world):
        (k0, k1), (q0, q1) = head_shard(hq, hkv, r, world)
        kv_seen += list(range(k0, k1))
        q_seen += list(range(q0, q1))
        for h in range(q0, q1):               # every q head of the shard attends a local kv head
            assert k0 <= h // G < k1
    assert kv_seen == list(range(hkv)) and q_seen == list(range(hq))


def test_head_shard_rejects_bad_world():
    with pytest.raises(ValueError):
        head_shard(64, 8, 0, 3)


def test_lpt_partition_balance_determinism():
    import neo_inputs as ni
    ctx = ni.ctx_loguniform(5, 1024, 128, 16384)
    parts = lpt_assign(ctx, 8)
    allids = np.sort(np.concatenate(parts))
    assert np.array_equal(allids, np.arange(1024))
    loads = [int(ctx[p].sum()) for p in parts]
    assert max(loads) - min(loads) <= int(ctx.max())        # LPT bound
    assert max(loads) / (sum(loads) / 8) < 1.01
    again = lpt_assign(ctx, 8)
    assert all(np.array_equal(a, b) for a, b in zip(parts, again))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import neo_inputs as ni
    import oracle
    seed, hq, hkv = 77, 64, 8
    ctx = [5, 300, 17]
    (k0, k1), (q0, q1) = head_shard(hq, hkv, rank, world)
    outs = []
    for b, n in enumerate(ctx):
        q = ni.q_bits(seed, 0, [b], hq, 128, heads=np.arange(q0, q1))[0]
        k = ni.kv_bits(seed, 0, ni.KIND_K, b, 0, n, hkv, 128, heads=np.arange(k0, k1))
        v = ni.kv_bits(seed, 0, ni.KIND_V, b, 0, n, hkv, 128, heads=np.arange(k0, k1))
        outs.append(oracle.decode_attention(q, k, v, 1 / math.sqrt(128)))
    local = torch.from_numpy(np.stack(outs))                 # [B][Hq/N][D]
    full = gather_heads(local, world)
    # request sharding: LPT, results exchanged with all_gather_object
    parts = lpt_assign(np.array(ctx), world)
    mine = {}
    for b in parts[rank]:
        n = ctx[b]
        q = ni.q_bits(seed, 1, [int(b)], hq, 128)[0]
        k = ni.kv_bits(seed, 1, ni.KIND_K, int(b), 0, n, hkv, 128)
        v = ni.kv_bits(seed, 1, ni.KIND_V, int(b), 0, n, hkv, 128)
        mine[int(b)] = oracle.decode_attention(q, k, v, 1 / math.sqrt(128))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        np.save(os.path.join(result_dir, "heads.npy"), full.numpy())
        merged = {}
        for d in gathered:
            merged.update(d)
        np.save(os.path.join(result_dir, "reqs.npy"), np.stack([merged[b] for b in range(len(ctx))]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reassembly_matches_single_process(tmp_path):
    import neo_inputs as ni
    import oracle
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    heads = np.load(tmp_path / "heads.npy")
    reqs = np.load(tmp_path / "reqs.npy")
    seed, hq, hkv = 77, 64, 8
    for b, n in enumerate([5, 300, 17]):
        for layer, got in ((0, heads[b]), (1, reqs[b])):
            q = ni.q_bits(seed, layer, [b], hq, 128)[0]
            k = ni.kv_bits(seed, layer, ni.KIND_K, b, 0, n, hkv, 128)
            v = ni.kv_bits(seed, layer, ni.KIND_V, b, 0, n, hkv, 128)
            ref = oracle.decode_attention(q, k, v, 1 / math.sqrt(128))
            assert np.array_equal(got, ref)                   # bitwise: sharding changes nothing
