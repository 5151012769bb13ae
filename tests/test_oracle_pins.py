"""Pins for the fp64 oracle against things other than itself (SURVEY §8(c)
"What pins each part", items 1-6): closed forms, brute force in Decimal,
a library routine (torch SDPA in fp64), and invariants.  CPU only."""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest
import torch

import oracle
from neo_inputs import (KIND_K, KIND_V, VARIANT_SINK, bf16_bits_to_f64, f32_to_bf16_bits,
                        kv_bits, q_bits)

SEED = 0x4E454F


def rand_bits(rng, shape, scale=1.0):
    return f32_to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32))


def widen(b):
    return bf16_bits_to_f64(b)


# 1. a 1-token context returns v exactly
@pytest.mark.parametrize("hq,hkv", [(4, 4), (8, 2), (32, 8)])
def test_single_token_returns_v(hq, hkv):
    rng = np.random.default_rng(1)
    q = rand_bits(rng, (hq, 128))
    k = rand_bits(rng, (1, hkv, 128))
    v = rand_bits(rng, (1, hkv, 128))
    out = oracle.decode_attention(q, k, v, 1 / math.sqrt(128))
    G = hq // hkv
    for h in range(hq):
        assert np.array_equal(out[h], widen(v[0, h // G]))


# 2. identical keys give the mean of V
def test_identical_keys_give_mean_of_v():
    rng = np.random.default_rng(2)
    n, hkv, hq = 5000, 2, 8
    q = rand_bits(rng, (hq, 128))
    krow = rand_bits(rng, (1, hkv, 128))
    k = np.repeat(krow, n, axis=0)
    v = rand_bits(rng, (n, hkv, 128))
    out = oracle.decode_attention(q, k, v, 0.088)
    vm = widen(v).mean(axis=0)
    for h in range(hq):
        np.testing.assert_allclose(out[h], vm[h // 4], rtol=0, atol=1e-13)


# 3. one-hot dominant score returns that row: q = 1, k_j = 4, others 0 => s_j = 45.25
def test_one_hot_dominant_score():
    n, j = 16384, 9876
    q = np.full((1, 128), 0x3F80, dtype=np.uint16)            # bf16 1.0
    k = np.zeros((n, 1, 128), dtype=np.uint16)
    k[j] = 0x4080                                              # bf16 4.0
    rng = np.random.default_rng(3)
    v = rand_bits(rng, (n, 1, 128))
    out = oracle.decode_attention(q, k, v, 1 / math.sqrt(128))
    # remaining weight: (n-1) e^{-45.25} ~ 3.6e-16 of the total
    np.testing.assert_allclose(out[0], widen(v[j, 0]), rtol=0, atol=1e-14)


# 4. constant V, any keys -> that constant
def test_constant_v():
    rng = np.random.default_rng(4)
    n = 777
    q = rand_bits(rng, (4, 128), 3.0)
    k = rand_bits(rng, (n, 1, 128))
    vrow = rand_bits(rng, (1, 1, 128))
    v = np.repeat(vrow, n, axis=0)
    out = oracle.decode_attention(q, k, v, 1 / math.sqrt(128))
    for h in range(4):
        np.testing.assert_allclose(out[h], widen(vrow[0, 0]), rtol=1e-14, atol=1e-15)


# 5. brute force: Decimal at 50 digits, naive softmax without max subtraction
def _decimal_attention(q, k, v, scale, G):
    getcontext().prec = 50
    hq, d = q.shape
    n = k.shape[0]
    out = np.zeros((hq, d))
    sc = Decimal(scale)
    for h in range(hq):
        g = h // G
        e = []
        for t in range(n):
            s = sum(Decimal(float(q[h, i])) * Decimal(float(k[t, g, i])) for i in range(d))
            e.append((s * sc).exp())
        den = sum(e)
        for i in range(d):
            out[h, i] = float(sum(e[t] * Decimal(float(v[t, g, i])) for t in range(n)) / den)
    return out


@pytest.mark.parametrize("trial", range(12))
def test_brute_force_decimal(trial):
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(1, 9))
    d = int(rng.integers(1, 9))
    hkv = int(rng.integers(1, 3))
    G = int(rng.choice([1, 2, 4]))
    hq = hkv * G
    q = rand_bits(rng, (hq, d), 2.0)
    k = rand_bits(rng, (n, hkv, d), 2.0)
    v = rand_bits(rng, (n, hkv, d))
    scale = float(np.float32(1 / math.sqrt(d)))
    got = oracle.decode_attention(q, k, v, scale)
    ref = _decimal_attention(widen(q), widen(k), widen(v), scale, G)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


# library routine: torch SDPA in fp64 with HF repeat_kv (g = h // G) semantics
@pytest.mark.parametrize("hq,hkv,n", [(32, 8, 300), (64, 8, 129), (32, 32, 17), (8, 1, 1000)])
def test_against_torch_sdpa_fp64(hq, hkv, n):
    rng = np.random.default_rng(hq * 1000 + n)
    q = rand_bits(rng, (hq, 128))
    k = rand_bits(rng, (n, hkv, 128))
    v = rand_bits(rng, (n, hkv, 128))
    scale = 1 / math.sqrt(128)
    got = oracle.decode_attention(q, k, v, scale)
    G = hq // hkv
    tq = torch.from_numpy(widen(q))[:, None, :]                       # [Hq][1][D]
    tk = torch.from_numpy(widen(k)).permute(1, 0, 2).repeat_interleave(G, 0)   # [Hq][n][D]
    tv = torch.from_numpy(widen(v)).permute(1, 0, 2).repeat_interleave(G, 0)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, scale=scale)[:, 0].numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)


# 6a. token-permutation invariance
def test_token_permutation_invariance():
    rng = np.random.default_rng(6)
    n = 1000
    q = rand_bits(rng, (8, 128), 2.0)
    k = rand_bits(rng, (n, 2, 128))
    v = rand_bits(rng, (n, 2, 128))
    perm = rng.permutation(n)
    a = oracle.decode_attention(q, k, v, 0.09)
    b = oracle.decode_attention(q, k[perm], v[perm], 0.09)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


# 6b. weights are non-negative and sum to 1
def test_weights_sum_to_one():
    rng = np.random.default_rng(7)
    q = rand_bits(rng, (8, 128), 8.0)
    k = rand_bits(rng, (513, 2, 128))
    w = oracle.softmax_weights(q, k, 1 / math.sqrt(128))
    assert (w >= 0).all()
    np.testing.assert_allclose(w.sum(axis=1), 1.0, rtol=0, atol=1e-12)


# 6c. partition independence + merge identity / commutativity
def test_partition_independence_and_merge():
    rng = np.random.default_rng(8)
    n, hq, hkv = 2000, 8, 2
    q = rand_bits(rng, (hq, 128), 4.0)
    k = rand_bits(rng, (n, hkv, 128))
    v = rand_bits(rng, (n, hkv, 128))
    scale = 1 / math.sqrt(128)
    full = oracle.decode_attention(q, k, v, scale)
    for trial in range(5):
        cuts = np.sort(rng.choice(np.arange(1, n), size=int(rng.integers(1, 12)), replace=False))
        bounds = [0, *cuts.tolist(), n]
        for h in (0, 5):
            parts = [oracle.partial(q, k, v, h, bounds[i], bounds[i + 1], scale)
                     for i in range(len(bounds) - 1)]
            ms, ls, accs = zip(*parts)
            merged = oracle.merge(ms, ls, np.stack(accs))
            np.testing.assert_allclose(merged, full[h], rtol=1e-12, atol=1e-14)
            perm = rng.permutation(len(parts))
            merged_p = oracle.merge(np.array(ms)[perm], np.array(ls)[perm], np.stack(accs)[perm])
            np.testing.assert_allclose(merged_p, merged, rtol=1e-12, atol=1e-14)
    # identity: a single partial returns acc / l
    m, l, acc = oracle.partial(q, k, v, 3, 0, n, scale)
    np.testing.assert_allclose(oracle.merge([m], [l], acc[None]), acc / l, rtol=0, atol=0)
    np.testing.assert_allclose(acc / l, full[3], rtol=1e-13, atol=1e-15)


# 6d. GQA mapping g = floor(h / G) via KV heads with disjoint supports
@pytest.mark.parametrize("G", [2, 4, 8])
def test_gqa_disjoint_supports(G):
    rng = np.random.default_rng(9 + G)
    hkv, d, n = 4, 128, 64
    hq = hkv * G
    blk = d // hkv
    q = rand_bits(rng, (hq, d))
    k = rand_bits(rng, (n, hkv, d))
    v = np.zeros((n, hkv, d), dtype=np.uint16)
    for g in range(hkv):
        v[:, g, g * blk:(g + 1) * blk] = rand_bits(rng, (n, blk))
    out = oracle.decode_attention(q, k, v, 0.1)
    for h in range(hq):
        g = h // G
        support = np.nonzero(out[h])[0]
        assert support.min() >= g * blk and support.max() < (g + 1) * blk
        single = oracle.decode_attention(q[h:h + 1], k[:, g:g + 1], v[:, g:g + 1], 0.1)
        np.testing.assert_array_equal(out[h], single[0])


def test_empty_context_is_zero():
    q = np.full((4, 128), 0x3F80, dtype=np.uint16)
    out = oracle.decode_attention(q, np.zeros((0, 1, 128), np.uint16), np.zeros((0, 1, 128), np.uint16), 0.1)
    assert (out == 0).all()


def test_shape_error():
    q = np.zeros((3, 128), dtype=np.uint16)
    k = np.zeros((4, 2, 128), dtype=np.uint16)
    with pytest.raises(ValueError):
        oracle.decode_attention(q, k, k, 0.1)


# generator-built sink inputs: the dominant token-0 logit makes the output close to v_0
def test_sink_variant_dominates():
    hq, hkv, n = 32, 8, 300
    q = q_bits(SEED, 0, [3], hq, 128)[0]
    k = kv_bits(SEED, 0, KIND_K, 3, 0, n, hkv, 128, variant=VARIANT_SINK, hq_total=hq)
    v = kv_bits(SEED, 0, KIND_V, 3, 0, n, hkv, 128)
    w = oracle.softmax_weights(q, k, 1 / math.sqrt(128))
    assert np.median(w[:, 0]) > 0.5


# swap definition: brute-force loop over every element vs the numpy indexing
def test_gather_pages_definition():
    rng = np.random.default_rng(11)
    L, NP, H, P, D = 3, 10, 2, 4, 8
    pool = rng.integers(0, 65535, size=(L, 2, NP, H, P, D), dtype=np.uint16)
    ids = [7, 2, 9]
    rec = oracle.gather_pages(pool, ids, 1, 3)
    assert rec.shape == (3, 2, 2, H, P, D)
    for i, pid in enumerate(ids):
        for l in range(1, 3):
            for kv in range(2):
                assert np.array_equal(rec[i, l - 1, kv], pool[l, kv, pid])
    host = rng.integers(0, 65535, size=(6, L, 2, H, P, D), dtype=np.uint16)
    hr = oracle.host_record(host, [5, 0], 0, 2)
    assert np.array_equal(hr[0], host[5, 0:2]) and np.array_equal(hr[1], host[0, 0:2])


# ---- RoPE oracle pins (oracle/rope.py)
def test_rope_identity_at_position_zero():
    from oracle import rope as orope
    rng = np.random.default_rng(20)
    x = rng.standard_normal((4, 128))
    assert np.array_equal(orope.rope(x, 0, orope.llama_inv_freq()), x)


def test_rope_preserves_pair_norms_and_matches_complex_form():
    from oracle import rope as orope
    rng = np.random.default_rng(21)
    x = rng.standard_normal((3, 128))
    f = orope.llama_inv_freq()
    for pos in (1, 17, 4095, 16383):
        y = orope.rope(x, pos, f)
        n0 = x[:, :64] ** 2 + x[:, 64:] ** 2
        n1 = y[:, :64] ** 2 + y[:, 64:] ** 2
        np.testing.assert_allclose(n1, n0, rtol=1e-12)
        z = (x[:, :64] + 1j * x[:, 64:]) * np.exp(1j * pos * f.astype(np.float64))
        np.testing.assert_allclose(y, np.concatenate([z.real, z.imag], axis=1), rtol=1e-12, atol=1e-12)


def test_rope_relative_position_property():
    """<R_m q, R_n k> = <q, R_{n-m} k>: attention scores depend only on n - m."""
    from oracle import rope as orope
    rng = np.random.default_rng(22)
    q, k = rng.standard_normal(128), rng.standard_normal(128)
    f = orope.llama_inv_freq()
    for m, n in ((3, 10), (100, 5000), (7000, 7001)):
        lhs = orope.rope(q, m, f) @ orope.rope(k, n, f)
        rhs = q @ orope.rope(k, n - m, f)
        assert abs(lhs - rhs) <= 1e-9 * (abs(rhs) + np.linalg.norm(q) * np.linalg.norm(k))


# ---- prefill oracle pins (oracle.prefill_attention)
@pytest.mark.parametrize("n,n_q,hq,hkv", [(300, 300, 32, 8), (500, 129, 8, 2), (64, 1, 4, 4), (200, 77, 16, 1)])
def test_prefill_against_torch_sdpa_causal_fp64(n, n_q, hq, hkv):
    """Library routine: torch SDPA in fp64 with an explicit bottom-right causal mask."""
    rng = np.random.default_rng(n * 7 + n_q)
    q = rand_bits(rng, (n_q, hq, 128), 2.0)
    k = rand_bits(rng, (n, hkv, 128))
    v = rand_bits(rng, (n, hkv, 128))
    scale = 1 / math.sqrt(128)
    got = oracle.prefill_attention(q, k, v, scale)
    G = hq // hkv
    tq = torch.from_numpy(widen(q)).permute(1, 0, 2)                                  # [Hq][n_q][D]
    tk = torch.from_numpy(widen(k)).permute(1, 0, 2).repeat_interleave(G, 0)          # [Hq][n][D]
    tv = torch.from_numpy(widen(v)).permute(1, 0, 2).repeat_interleave(G, 0)
    mask = torch.arange(n)[None, :] <= (n - n_q + torch.arange(n_q))[:, None]        # [n_q][n]
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=scale)
    np.testing.assert_allclose(got, ref.permute(1, 0, 2).numpy(), rtol=1e-12, atol=1e-13)


def test_prefill_first_row_of_full_prompt_is_v0():
    """A whole-prompt prefill: row 0 sees only token 0, so its output is V[0] exactly."""
    rng = np.random.default_rng(23)
    q = rand_bits(rng, (40, 8, 128), 3.0)
    k = rand_bits(rng, (40, 2, 128))
    v = rand_bits(rng, (40, 2, 128))
    out = oracle.prefill_attention(q, k, v, 0.1)
    for h in range(8):
        assert np.array_equal(out[0, h], widen(v[0, h // 4]))


def test_prefill_is_causal():
    """Changing K/V of tokens after a row's position leaves that row bit-identical,
    and changes the rows that can see them."""
    rng = np.random.default_rng(24)
    n, n_q = 120, 50
    q = rand_bits(rng, (n_q, 8, 128), 2.0)
    k = rand_bits(rng, (n, 2, 128))
    v = rand_bits(rng, (n, 2, 128))
    a = oracle.prefill_attention(q, k, v, 0.09)
    cut = n - n_q + 20                                        # rows 0..20 see tokens < cut + 1
    k2, v2 = k.copy(), v.copy()
    k2[cut + 1:] = rand_bits(rng, k2[cut + 1:].shape)
    v2[cut + 1:] = rand_bits(rng, v2[cut + 1:].shape)
    b = oracle.prefill_attention(q, k2, v2, 0.09)
    assert np.array_equal(a[:21], b[:21])
    assert not np.allclose(a[21:], b[21:])


@pytest.mark.parametrize("trial", range(4))
def test_prefill_brute_force_decimal(trial):
    rng = np.random.default_rng(300 + trial)
    n = int(rng.integers(1, 7))
    n_q = int(rng.integers(1, n + 1))
    hkv, G, d = 1, int(rng.choice([1, 2])), int(rng.integers(1, 6))
    q = rand_bits(rng, (n_q, hkv * G, d), 2.0)
    k = rand_bits(rng, (n, hkv, d), 2.0)
    v = rand_bits(rng, (n, hkv, d))
    scale = float(np.float32(1 / math.sqrt(d)))
    got = oracle.prefill_attention(q, k, v, scale)
    for i in range(n_q):
        p = n - n_q + i + 1
        ref = _decimal_attention(widen(q[i]), widen(k[:p]), widen(v[:p]), scale, G)
        np.testing.assert_allclose(got[i], ref, rtol=1e-13, atol=1e-15)


# ---- batch driver (oracle_decode_attention_batch): it produces every cpu_baseline
# and --impl reference number, so it is pinned on its own: against fp64 torch SDPA
# request by request (a library routine), and bit for bit against the single-request
# definition over ragged offsets and any thread count (an offset or stride bug in the
# packing shows up as a wrong request, a thread-split bug as a missing one).
def _ragged_batch(rng, lens, hq, hkv, scale_q=2.0):
    q = rand_bits(rng, (len(lens), hq, 128), scale_q)
    ks = [rand_bits(rng, (n, hkv, 128)) for n in lens]
    vs = [rand_bits(rng, (n, hkv, 128)) for n in lens]
    return q, ks, vs


@pytest.mark.parametrize("nthreads", [1, 3, 16])
def test_batch_equals_single_request_bitwise(nthreads):
    rng = np.random.default_rng(400 + nthreads)
    lens = [1, 17, 300, 2, 129, 16, 1000, 5, 64, 33, 7]
    q, ks, vs = _ragged_batch(rng, lens, 32, 8)
    scale = 1 / math.sqrt(128)
    got = oracle.decode_attention_batch(q, ks, vs, scale, nthreads=nthreads)
    assert got.shape == (len(lens), 32, 128)
    for b in range(len(lens)):
        assert np.array_equal(got[b], oracle.decode_attention(q[b], ks[b], vs[b], scale)), b


@pytest.mark.parametrize("hq,hkv", [(32, 8), (64, 8), (8, 8)])
def test_batch_against_torch_sdpa_fp64(hq, hkv):
    rng = np.random.default_rng(hq + 7 * hkv)
    lens = [3, 250, 1, 97, 512]
    q, ks, vs = _ragged_batch(rng, lens, hq, hkv)
    scale = 1 / math.sqrt(128)
    got = oracle.decode_attention_batch(q, ks, vs, scale, nthreads=4)
    G = hq // hkv
    for b, n in enumerate(lens):
        tq = torch.from_numpy(widen(q[b]))[:, None, :]
        tk = torch.from_numpy(widen(ks[b])).permute(1, 0, 2).repeat_interleave(G, 0)
        tv = torch.from_numpy(widen(vs[b])).permute(1, 0, 2).repeat_interleave(G, 0)
        ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, scale=scale)[:, 0].numpy()
        np.testing.assert_allclose(got[b], ref, rtol=1e-12, atol=1e-13)


def test_batch_more_threads_than_requests():
    rng = np.random.default_rng(410)
    q, ks, vs = _ragged_batch(rng, [40, 9], 8, 2)
    got = oracle.decode_attention_batch(q, ks, vs, 0.1, nthreads=64)
    for b in range(2):
        assert np.array_equal(got[b], oracle.decode_attention(q[b], ks[b], vs[b], 0.1))


# ---- softmax weights (oracle_softmax_weights), beyond "sum to 1": a wrong scale,
# a wrong GQA group or a token offset each change the weights themselves.
@pytest.mark.parametrize("hq,hkv,n", [(32, 8, 300), (8, 1, 77), (16, 16, 5), (64, 8, 1)])
def test_softmax_weights_against_torch_softmax_fp64(hq, hkv, n):
    rng = np.random.default_rng(500 + n)
    q = rand_bits(rng, (hq, 128), 3.0)
    k = rand_bits(rng, (n, hkv, 128))
    scale = float(np.float32(1 / math.sqrt(128)))
    w = oracle.softmax_weights(q, k, scale)
    G = hq // hkv
    tq = torch.from_numpy(widen(q))                                                    # [Hq][D]
    tk = torch.from_numpy(widen(k)).permute(1, 0, 2).repeat_interleave(G, 0)          # [Hq][n][D]
    ref = torch.softmax(scale * torch.einsum("hd,htd->ht", tq, tk), dim=-1).numpy()
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-15)


def test_softmax_weights_times_v_is_decode_attention():
    rng = np.random.default_rng(510)
    hq, hkv, n = 32, 8, 700
    q = rand_bits(rng, (hq, 128), 4.0)
    k = rand_bits(rng, (n, hkv, 128))
    v = rand_bits(rng, (n, hkv, 128))
    scale = 1 / math.sqrt(128)
    w = oracle.softmax_weights(q, k, scale)
    out = oracle.decode_attention(q, k, v, scale)
    G = hq // hkv
    vv = widen(v)
    for h in range(hq):
        np.testing.assert_allclose(w[h] @ vv[:, h // G], out[h], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("trial", range(6))
def test_softmax_weights_brute_force_decimal(trial):
    getcontext().prec = 50
    rng = np.random.default_rng(520 + trial)
    n, d = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    hkv, G = int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
    q = rand_bits(rng, (hkv * G, d), 2.0)
    k = rand_bits(rng, (n, hkv, d), 2.0)
    scale = float(np.float32(1 / math.sqrt(d)))
    w = oracle.softmax_weights(q, k, scale)
    qf, kf = widen(q), widen(k)
    for h in range(hkv * G):
        e = [(Decimal(scale) * sum(Decimal(float(qf[h, i])) * Decimal(float(kf[t, h // G, i]))
                                   for i in range(d))).exp() for t in range(n)]
        den = sum(e)
        np.testing.assert_allclose(w[h], [float(x / den) for x in e], rtol=1e-13, atol=1e-16)


# ---- flash-decoding task statistics (oracle_partial) written out with torch fp64 ops
def test_partial_statistics_against_torch_fp64():
    rng = np.random.default_rng(530)
    hq, hkv, n = 16, 4, 900
    q = rand_bits(rng, (hq, 128), 3.0)
    k = rand_bits(rng, (n, hkv, 128))
    v = rand_bits(rng, (n, hkv, 128))
    scale = float(np.float32(1 / math.sqrt(128)))
    G = hq // hkv
    for h, t0, t1 in ((0, 0, n), (5, 100, 101), (11, 333, 777), (15, 899, 900)):
        m, l, acc = oracle.partial(q, k, v, h, t0, t1, scale)
        s = scale * (torch.from_numpy(widen(k[t0:t1, h // G])) @ torch.from_numpy(widen(q[h])))
        e = torch.exp(s - s.max())
        assert m == pytest.approx(float(s.max()), rel=1e-14, abs=1e-14)
        assert l == pytest.approx(float(e.sum()), rel=1e-13)
        np.testing.assert_allclose(acc, (e[:, None] * torch.from_numpy(widen(v[t0:t1, h // G]))).sum(0).numpy(),
                                   rtol=1e-12, atol=1e-12)


def test_merge_closed_form_two_parts():
    """Two partials with m_1 = m_2 + ln 2 and equal l, acc: the first counts twice
    as much, so out = (2 a_1 + a_2) / (2 l + l)."""
    a1, a2 = np.arange(4.0), np.array([1.0, -1.0, 0.5, 3.0])
    out = oracle.merge([0.5 + math.log(2.0), 0.5], [3.0, 3.0], np.stack([a1, a2]))
    np.testing.assert_allclose(out, (2 * a1 + a2) / 9.0, rtol=1e-15, atol=1e-16)
