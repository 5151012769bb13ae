"""Pins for the seeded input generator (neo_inputs): published splitmix64
outputs, bf16 round-to-nearest-even against torch, distribution moments, and
the metadata recipes (P:364 uniform lengths, S:120 integer rounding)."""
import numpy as np
import torch

import neo_inputs as ni


def test_splitmix64_reference_outputs():
    # Reference splitmix64 stream from state 0 (Vigna's splitmix64.c): the
    # generator returns splitmix64(k * gamma) for k = 0, 1, 2, ... in our form.
    expected = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    states = np.array([(k * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF for k in range(4)], dtype=np.uint64)
    got = ni.splitmix64(states)
    assert [int(x) for x in got] == expected


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    f = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10,
                        np.array([1.00390625, 1.01171875, -1.00390625, 0.0, -0.0, 3.0e-39], np.float32)])
    ours = ni.f32_to_bf16_bits(f)
    ref = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_counter_values_moments_and_determinism():
    idx = np.arange(1 << 18, dtype=np.uint64)
    a = ni.counter_bits(ni.DEFAULT_SEED, ni.tensor_id(ni.KIND_K, 3), idx)
    b = ni.counter_bits(ni.DEFAULT_SEED, ni.tensor_id(ni.KIND_K, 3), idx)
    assert np.array_equal(a, b)
    x = ni.bf16_bits_to_f64(a)
    assert abs(x.mean()) < 0.01
    assert abs(x.std() - 1.1547) < 0.01          # 4 uniform 16-bit sums: sqrt(4/12)*2 = 1.1547
    assert np.abs(x).max() <= 131070 / 32768
    c = ni.counter_bits(ni.DEFAULT_SEED, ni.tensor_id(ni.KIND_V, 3), idx)
    assert not np.array_equal(a, c)


def test_kv_bits_independent_of_slicing():
    full = ni.kv_bits(7, 2, ni.KIND_V, 5, 0, 40, 8, 128)
    part = ni.kv_bits(7, 2, ni.KIND_V, 5, 16, 40, 8, 128, heads=[3, 4])
    assert np.array_equal(full[16:, 3:5], part)
    q = ni.q_bits(7, 2, [0, 1, 2], 32, 128)
    assert np.array_equal(q[1:2, 8:16], ni.q_bits(7, 2, [1], 32, 128, heads=np.arange(8, 16)))


def test_peaked_is_times_eight():
    q = ni.q_bits(7, 0, [0], 8, 128)
    qp = ni.q_bits(7, 0, [0], 8, 128, variant=ni.VARIANT_PEAKED)
    assert np.array_equal(ni.bf16_bits_to_f64(qp), 8 * ni.bf16_bits_to_f64(q))


def test_sink_row():
    hq, hkv = 32, 8
    k = ni.kv_bits(7, 1, ni.KIND_K, 2, 0, 3, hkv, 128, variant=ni.VARIANT_SINK, hq_total=hq)
    q = ni.bf16_bits_to_f64(ni.q_bits(7, 1, [2], hq, 128))[0]
    for g in range(hkv):
        expect = np.where(q[g * 4:(g + 1) * 4].sum(axis=0) >= 0, 4.0, -4.0)
        assert np.array_equal(ni.bf16_bits_to_f64(k[0, g]), expect)
    plain = ni.kv_bits(7, 1, ni.KIND_K, 2, 0, 3, hkv, 128)
    assert np.array_equal(plain[1:], k[1:])


def test_ctx_uniform_bounds():
    c = ni.ctx_uniform(1, 10000, 1024)
    assert c.min() == 922 and c.max() == 1126            # [ceil(921.6), floor(1126.4)]
    assert np.array_equal(c, ni.ctx_uniform(1, 10000, 1024))
    c = ni.ctx_uniform(2, 5000, 2048)
    assert c.min() >= 1844 and c.max() <= 2252


def test_ctx_loguniform_and_lognormal():
    c = ni.ctx_loguniform(3, 20000, 128, 16384)
    assert c.min() >= 128 and c.max() <= 16384
    assert 3000 < c.mean() < 3700                        # E = (16384-128)/ln(128) ~ 3350
    c = ni.ctx_lognormal(3, 20000, 1024, 0.75, 16, 8192)
    assert c.min() >= 16 and c.max() <= 8192 and 900 < np.median(c) < 1150


def test_block_tables_are_a_scattered_partition():
    ctx = np.array([1, 16, 17, 100, 0], dtype=np.int32)
    table, npages = ni.block_tables(5, ctx, 16, num_pages=64)
    need = ni.pages_needed(ctx, 16)
    used = np.concatenate([table[i, :need[i]] for i in range(len(ctx))])
    assert len(set(used.tolist())) == len(used) == need.sum()
    assert used.max() < 64 and used.min() >= 0
    for i in range(len(ctx)):
        assert (table[i, need[i]:] == -1).all()


def test_c_generator_matches_numpy():
    rng = np.random.default_rng(5)
    for trial in range(20):
        hkv = int(rng.choice([1, 2, 8, 32]))
        G = int(rng.choice([1, 4, 8]))
        hq = hkv * G
        b = int(rng.integers(0, 1024))
        t0 = int(rng.integers(0, 50))
        t1 = t0 + int(rng.integers(1, 40))
        layer = int(rng.integers(0, 80))
        variant = int(rng.integers(0, 4))
        g0 = int(rng.integers(0, hkv))
        heads = np.arange(g0, hkv)
        for kind in (ni.KIND_K, ni.KIND_V):
            a = ni.kv_bits(11, layer, kind, b, t0, t1, hkv, 128, heads=heads, variant=variant, hq_total=hq)
            c = ni.kv_bits(11, layer, kind, b, t0, t1, hkv, 128, heads=heads, variant=variant, hq_total=hq,
                           use_c=False)
            assert np.array_equal(a, c)
        if t0 == 0 or True:
            a = ni.kv_bits(11, layer, ni.KIND_K, b, 0, 3, hkv, 128, variant=variant, hq_total=hq)
            c = ni.kv_bits(11, layer, ni.KIND_K, b, 0, 3, hkv, 128, variant=variant, hq_total=hq, use_c=False)
            assert np.array_equal(a, c)
        qa = ni.q_bits(11, layer, [b, b + 1], hq, 128, heads=np.arange(G, hq), variant=variant)
        qc = ni.q_bits(11, layer, [b, b + 1], hq, 128, heads=np.arange(G, hq), variant=variant, use_c=False)
        assert np.array_equal(qa, qc)
