"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the a0 planner's chunk from the host lengths, device-generated inputs,
scattered block tables), and at the library-default chunk: sampled requests of sampled layers are checked one by one against the
fp64 oracle, and every output row is checked to be finite.  Head-sharded (c4)
and request-sharded (c5) shards are checked the same way on their slice."""
import math

import numpy as np
import pytest

from harness import within_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def run_and_sample(wl, layers, n_samples, rng, planned=True, **kw):
    import torch

    import oracle
    import neo_inputs as ni
    from neo_inputs.gpu import GpuBatch
    from paper_2411_01142_b200 import neo
    gb = GpuBatch(wl, layers=max(layers) + 1, **kw)
    C = neo.plan_chunk(gb.ctx, gb.hkv, gb.P) if planned else 0
    worst = 0.0
    for layer in layers:
        k, v = gb.layer(layer)
        out = neo.decode_attn(gb.q[layer], k, v, gb.block_table, gb.seq_lens, gb.max_seq_len, chunk_tokens=C)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
        picks = set(rng.choice(gb.B, size=min(n_samples, gb.B), replace=False).tolist())
        picks |= {int(np.argmax(gb.ctx)), int(np.argmin(gb.ctx))}          # longest and shortest
        for b in sorted(picks):
            q, kb, vb = gb.oracle_inputs(b, layer)
            ref = oracle.decode_attention(q, kb, vb, np.float32(1 / math.sqrt(128)))
            got = ni.bf16_bits_to_f64(out[b].view(torch.int16).cpu().numpy().view(np.uint16))
            ok, r = within_tol(got, ref)
            worst = max(worst, r)
            assert ok, f"{wl.name} layer {layer} request {b} ctx {gb.ctx[b]} err/tol {r:.3f}"
    del gb
    torch.cuda.empty_cache()
    return worst


@pytest.mark.parametrize("name,layers,n", [("c1", [0], 4), ("c2", [0, 31], 12), ("c2s", [5], 12),
                                           ("c3", [0, 17], 8), ("c4", [0, 3], 10), ("c5", [0], 12)])
def test_fullsize_sampled(name, layers, n):
    from neo_inputs.workloads import WORKLOADS
    rng = np.random.default_rng(hash(name) % 1000)
    w = run_and_sample(WORKLOADS[name], layers, n, rng)
    print(f"{name}: worst err/tol {w:.3f}")


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_fullsize_sampled_default_chunk(name):
    from neo_inputs.workloads import WORKLOADS
    rng = np.random.default_rng(7 + hash(name) % 1000)
    run_and_sample(WORKLOADS[name], [2], 8, rng, planned=False)


@pytest.mark.parametrize("world", [2, 8])
def test_fullsize_head_shard_c4(world):
    from neo_inputs.workloads import WORKLOADS
    from paper_2411_01142_b200.shard import head_shard
    wl = WORKLOADS["c4"]
    rng = np.random.default_rng(world)
    for rank in (0, world - 1):
        kvh, qh = head_shard(wl.hq, wl.hkv, rank, world)
        run_and_sample(wl, [1], 6, rng, kv_heads=kvh, q_heads=qh)


def test_fullsize_request_shard_c5():
    from neo_inputs.workloads import WORKLOADS
    from paper_2411_01142_b200.shard import lpt_assign
    wl = WORKLOADS["c5"]
    ctx = wl.contexts()
    parts = lpt_assign(ctx[:512], 8)                        # f = 0.5, 8 ranks
    rng = np.random.default_rng(5)
    run_and_sample(wl, [0], 6, rng, ctx=ctx, req_ids=parts[3])


@pytest.mark.parametrize("C", [256, -1, -4])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_head_shards_reassemble_bitwise(world, C):
    """KV-head shards (each rank's own heads, own pool),
    reassembled along heads, equal the unsharded output bit for bit at the same C."""
    import torch

    from neo_inputs.gpu import GpuBatch
    from neo_inputs.workloads import WORKLOADS
    from paper_2411_01142_b200 import neo
    from paper_2411_01142_b200.shard import head_shard
    wl = WORKLOADS["c4"]
    ctx = wl.contexts()[:96]
    full = GpuBatch(wl, ctx=ctx, layers=1)
    k, v = full.layer(0)
    ref = neo.decode_attn(full.q[0], k, v, full.block_table, full.seq_lens, full.max_seq_len, chunk_tokens=C)
    torch.cuda.synchronize()
    parts = []
    for rank in range(world):
        kvh, qh = head_shard(wl.hq, wl.hkv, rank, world)
        sh = GpuBatch(wl, ctx=ctx, layers=1, kv_heads=kvh, q_heads=qh)
        k, v = sh.layer(0)
        parts.append(neo.decode_attn(sh.q[0], k, v, sh.block_table, sh.seq_lens, sh.max_seq_len, chunk_tokens=C))
    torch.cuda.synchronize()
    got = torch.cat(parts, dim=1)
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("C", [128, -1, -2])
def test_request_shards_reassemble_bitwise(C):
    """Request (LPT) shards in their own pools and batches equal the unsharded
    output bit for bit: a request's result depends only on its inputs and C
    (for the grouped kernel, C = -1: on its own length)."""
    import torch

    from neo_inputs.gpu import GpuBatch
    from neo_inputs.workloads import WORKLOADS
    from paper_2411_01142_b200 import neo
    from paper_2411_01142_b200.shard import lpt_assign
    wl = WORKLOADS["c5"]
    ctx = wl.contexts()[:200]
    full = GpuBatch(wl, ctx=ctx, layers=1)
    k, v = full.layer(0)
    ref = neo.decode_attn(full.q[0], k, v, full.block_table, full.seq_lens, full.max_seq_len, chunk_tokens=C)
    torch.cuda.synchronize()
    for ids in lpt_assign(ctx, 4):
        sh = GpuBatch(wl, ctx=ctx, layers=1, req_ids=ids)
        k, v = sh.layer(0)
        out = neo.decode_attn(sh.q[0], k, v, sh.block_table, sh.seq_lens, sh.max_seq_len, chunk_tokens=C)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref[torch.from_numpy(ids).cuda()].view(torch.int16))
