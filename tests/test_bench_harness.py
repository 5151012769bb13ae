"""bench.py's multi-rank harness on CPU: the rank plans
cover every unit exactly once, and under gloo world size 2 the aggregation
(MAX time, SUM bytes, the head-sharding token rule, per-rank imbalance) and the
all-gather + permute reassembly of head shards give the single-process result.
The first multi-GPU run then cannot fail on harness logic."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from neo_inputs.workloads import WORKLOADS


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_shard_plans_cover_units_once(cfg, world):
    wl = WORKLOADS[cfg]
    plans = [bench.shard_plan(wl, r, world, 0.75) for r in range(world)]
    if cfg == "c4":                        # KV-head TP: full batch on every rank, heads partitioned
        kv = sum((list(range(*p[2])) for p in plans), [])
        qh = sum((list(range(*p[3])) for p in plans), [])
        assert kv == list(range(wl.hkv)) and qh == list(range(wl.hq))
        assert all(p[1] is None and np.array_equal(p[0], wl.contexts()) for p in plans)
        assert all(p[4] == "strong" for p in plans)
        return
    if cfg == "c5":                        # LPT over the GPU-resident first f*1024 requests
        ids = np.sort(np.concatenate([p[1] for p in plans]))
        assert np.array_equal(ids, np.arange(int(round(0.75 * wl.batch))))
        return
    if world == 1:
        assert plans[0][1] is None and plans[0][4] == "weak"
        return
    ctx = plans[0][0]
    assert len(ctx) == wl.batch * world and all(np.array_equal(p[0], ctx) for p in plans)
    ids = np.concatenate([p[1] for p in plans])
    assert np.array_equal(np.sort(ids), np.arange(wl.batch * world))     # weak: disjoint batches


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    # aggregation: rank r took (r + 1) seconds for 3 steps, read (r + 1) * 1e9 bytes, attended 100 * (r + 1) tokens
    for head_sharded in (False, True):
        res[head_sharded] = bench.aggregate_ranks(float(rank + 1), (rank + 1) * 1e9, 100.0 * (rank + 1), 3, world,
                                                  head_sharded=head_sharded, dist=dist, device="cpu")
    # reassembly of head shards (c4-like: 64 q heads / 8 kv heads, tiny contexts) through the oracle
    import neo_inputs as ni
    import oracle
    from paper_2411_01142_b200.shard import head_shard
    seed, hq, hkv, ctx = 91, 64, 8, [3, 40]
    (k0, k1), (q0, q1) = head_shard(hq, hkv, rank, world)
    outs = []
    for b, n in enumerate(ctx):
        q = ni.q_bits(seed, 0, [b], hq, 128, heads=np.arange(q0, q1))[0]
        k = ni.kv_bits(seed, 0, ni.KIND_K, b, 0, n, hkv, 128, heads=np.arange(k0, k1))
        v = ni.kv_bits(seed, 0, ni.KIND_V, b, 0, n, hkv, 128, heads=np.arange(k0, k1))
        outs.append(oracle.decode_attention(q, k, v, 1 / math.sqrt(128)))
    local = torch.from_numpy(np.stack(outs))                        # [B][Hq/N][D]
    gbuf = torch.empty((world,) + tuple(local.shape), dtype=local.dtype)
    dist.all_gather_into_tensor(gbuf.view(-1), local.contiguous().view(-1))
    full = torch.empty((len(ctx), hq, 128), dtype=local.dtype)
    bench.reassemble_heads_into(full, gbuf)
    if rank == 0:
        torch.save({"agg": res, "full": full}, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_aggregation_and_reassembly(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, start_method="spawn")
    r = torch.load(tmp_path / "res.pt", weights_only=False)
    t, kv, tok, per = r["agg"][False]
    assert t == 2.0 and kv == 3e9 and tok == 300.0                  # MAX time, SUM bytes, SUM tokens
    assert per == pytest.approx([1e3 / 3, 2e3 / 3])                  # ms per step of each rank
    assert bench.rank_imbalance(per) == pytest.approx(2 / 1.5, abs=1e-4)
    t, kv, tok, per = r["agg"][True]
    assert t == 2.0 and kv == 3e9 and tok == 100.0                   # head sharding: tokens counted once
    import neo_inputs as ni
    import oracle
    seed, hq, hkv = 91, 64, 8
    for b, n in enumerate([3, 40]):
        q = ni.q_bits(seed, 0, [b], hq, 128)[0]
        k = ni.kv_bits(seed, 0, ni.KIND_K, b, 0, n, hkv, 128)
        v = ni.kv_bits(seed, 0, ni.KIND_V, b, 0, n, hkv, 128)
        assert np.array_equal(r["full"][b].numpy(), oracle.decode_attention(q, k, v, 1 / math.sqrt(128)))


def test_single_rank_aggregation_is_identity():
    t, kv, tok, per = bench.aggregate_ranks(0.5, 7.0, 9.0, 4, 1, head_sharded=True)
    assert (t, kv, tok, per) == (0.5, 7.0, 9.0, None)


def test_batch_total_rules():
    from types import SimpleNamespace
    gb = SimpleNamespace(B=64)
    assert bench.batch_total(WORKLOADS["c4"], gb, 8, 1.0, None) == 64
    assert bench.batch_total(WORKLOADS["c5"], gb, 8, 0.25, np.zeros(1024)) == 256
    assert bench.batch_total(WORKLOADS["c2"], gb, 4, 1.0, None) == 256
