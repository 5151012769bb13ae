"""GPU parity of neo_decode_attn against the fp64 oracle (SURVEY §8(c) items
7-10 and 15's single-GPU part), through the C ABI.  Tolerance: the north
star's |gpu - ref| <= 2e-3 + 1e-2 |ref| elementwise; bit-exact where the
integer part (block table, masking, relocation) decides."""
import math

import numpy as np
import pytest

import neo_inputs as ni
from harness import Case, within_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def check_case(case, chunk=0, tag=""):
    out = case.run(chunk_tokens=chunk)
    got = case.out_f64(out)
    worst = 0.0
    for b in range(case.B):
        ok, ratio = within_tol(got[b], case.oracle(b))
        worst = max(worst, ratio)
        assert ok, f"{tag} b={b} ctx={case.ctx[b]} err/tol={ratio:.3f}"
    return out, worst


@pytest.mark.parametrize("hq,hkv", [(32, 32), (32, 8), (64, 8), (16, 8), (8, 1)])
@pytest.mark.parametrize("chunk", [0, 16, 64, 256, 512])
def test_parity_ragged(hq, hkv, chunk):
    ctx = [1, 15, 16, 17, 31, 32, 33, 127, 128, 129, 600, 1000]
    case = Case(ctx, hq, hkv, seed=1 + hq + hkv + chunk)
    check_case(case, chunk, f"G={hq // hkv} C={chunk}")


@pytest.mark.parametrize("hq,hkv", [(24, 8), (40, 8), (48, 8), (28, 4), (7, 1)])
@pytest.mark.parametrize("chunk", [16, 64, 512])
def test_parity_group_sizes_not_dividing_32(hq, hkv, chunk):
    """G in {3, 5, 6, 7} (e.g. 28 q / 4 kv heads): the combine's per-head
    statistics must not assume G divides the warp size."""
    ctx = [1, 16, 17, 129, 600, 1000, 2049]
    check_case(Case(ctx, hq, hkv, seed=13 + hq + chunk), chunk, f"G={hq // hkv} C={chunk}")


@pytest.mark.parametrize("chunk", [192, 320, 384, 448, 768, 1024])
def test_parity_planner_chunks(chunk):
    """Non-power-of-two chunks the a0 planner (neo_decode_attn_plan_chunk) picks,
    on contexts that end at, one past and one short of chunk boundaries."""
    ctx = [1, chunk - 1, chunk, chunk + 1, 2 * chunk + 17, 1844, 2252]
    case = Case(ctx, 64, 8, seed=11 + chunk)
    check_case(case, chunk, f"C={chunk}")


def test_parity_planned_chunk_c4_shard():
    """The chunk the planner picks for one kv-head of a c4-like batch, end to end."""
    from paper_2411_01142_b200 import neo
    rng = np.random.default_rng(8)
    ctx = rng.integers(1844, 2253, size=64)
    C = neo.plan_chunk(ctx, 1, 16)
    assert C in (-1, -2, -4) or (C % 16 == 0 and 16 <= C <= 1024)
    check_case(Case(ctx, 8, 1, seed=12), C, f"planned C={C}")


@pytest.mark.parametrize("P,chunk", [(32, 64), (32, 0), (64, 128), (32, 512)])
def test_parity_page_sizes(P, chunk):
    case = Case([1, 31, 32, 33, 95, 513, 700], 32, 8, P=P, seed=7 + P)
    check_case(case, chunk, f"P={P}")


def test_parity_padded_page_stride():
    # page-major style layout: pages 3x further apart than Hkv*P*D
    case = Case([5, 40, 300], 32, 8, page_stride=3 * 8 * 16 * 128, seed=11)
    check_case(case, 64)


@pytest.mark.parametrize("variant", [ni.VARIANT_PEAKED, ni.VARIANT_SINK, ni.VARIANT_PEAKED | ni.VARIANT_SINK])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (64, 8), (32, 32)])
def test_parity_variants(variant, hq, hkv):
    case = Case([1, 17, 250, 1100, 2049], hq, hkv, variant=variant, seed=21 + variant)
    for chunk in (0, 64):
        check_case(case, chunk, f"variant={variant}")


def test_parity_random_configs():
    """>= 500 random small configs (S:599 mirrored): ctx 1-600 incl. multiples of P
    and P+-1, G in {1,2,4,8}, shuffled block tables, C in {16, 64, 256, 512}."""
    rng = np.random.default_rng(599)
    worst = 0.0
    for trial in range(520):
        G = int(rng.choice([1, 2, 4, 8]))
        hkv = int(rng.choice([1, 2, 4, 8]))
        B = int(rng.integers(1, 4))
        P = int(rng.choice([16, 16, 32]))
        kind = rng.integers(0, 3)
        if kind == 0:
            ctx = rng.integers(1, 601, size=B)
        else:
            base = P * rng.integers(1, 600 // P + 1, size=B)
            ctx = np.clip(base + (rng.integers(-1, 2, size=B) if kind == 1 else 0), 1, 600)
        C = int(rng.choice([16, 64, 256, 512]))
        if C % P:
            C = P * max(1, C // P)
        case = Case(ctx, hkv * G, hkv, P=P, seed=1000 + trial, variant=int(rng.choice([0, 0, 1, 2])))
        _, r = check_case(case, C, f"trial {trial}")
        worst = max(worst, r)
    print(f"worst err/tol over random configs: {worst:.3f}")


def test_single_token_bitwise_v():
    case = Case([1, 1, 1], 32, 8, seed=5)
    out = case.run()
    got = case.out_f64(out)
    for b in range(3):
        for h in range(32):
            assert np.array_equal(got[b, h], ni.bf16_bits_to_f64(case.v_req[b][0, h // 4]))


def test_one_hot_dominant_bitwise():
    """q = 1, k_j = 4 (s_j = 45.25), other k = 0: output is v_j bit for bit."""
    import torch
    from paper_2411_01142_b200 import neo
    n, j = 16384, 9876
    case = Case([n], 8, 1, seed=6)
    k = case.k_dev.view(-1, 16, 128)             # [pages][P][D] (Hkv=1)
    k.zero_()
    table = case.table[0]
    k[table[j // 16], j % 16] = 4.0
    case.q_dev.fill_(1.0)
    for chunk in (0, 64, 512):
        out = case.run(chunk_tokens=chunk)
        got = case.out_f64(out)
        vj = ni.bf16_bits_to_f64(case.v_req[0][j, 0])
        for h in range(8):
            assert np.array_equal(got[0, h], vj), chunk


def test_identical_keys_mean_of_v():
    case = Case([3000], 32, 8, seed=8)
    k = case.k_dev
    kb = k[case.table[0, 0], :, 0:1, :].clone()          # token 0's K row for all heads
    k.copy_(kb.unsqueeze(0).expand(k.shape[0], -1, 16, -1))
    out = case.run()
    got = case.out_f64(out)
    vm = ni.bf16_bits_to_f64(case.v_req[0]).mean(axis=0)  # [Hkv][D]
    for h in range(32):
        ok, r = within_tol(got[0, h], vm[h // 4])
        assert ok, r


def test_relocation_and_poison_bitwise():
    """Moving physical pages (same logical order) and NaN in every slot the kernel
    must not read leave the output bitwise unchanged (items 9, 10)."""
    ctx = [1, 17, 100, 257, 1000]
    a = Case(ctx, 32, 8, seed=9, table_seed=1, tail="zero", fill_unused="zero", extra_pages=0)
    b = Case(ctx, 32, 8, seed=9, table_seed=2, tail="nan", fill_unused="nan", extra_pages=40)
    assert not np.array_equal(a.table, b.table)
    for chunk in (0, 16, 64, -1):
        import torch
        oa = a.run(chunk_tokens=chunk)
        ob = b.run(chunk_tokens=chunk)
        assert torch.isfinite(ob.float()).all()
        assert torch.equal(oa.view(torch.int16), ob.view(torch.int16))


def test_block_table_padding_ignored():
    import torch
    case = Case([20, 50], 32, 8, seed=12)
    bt = torch.full((2, case.max_blocks + 5), 12345678, dtype=torch.int32, device="cuda")
    bt[:, :case.max_blocks] = case.bt_dev
    bt[0, 2:] = -1                                  # entries past ceil(ctx/P) are never read
    base = case.run()
    from paper_2411_01142_b200 import neo
    out = neo.decode_attn(case.q_dev, case.k_dev, case.v_dev, bt, case.sl_dev, case.max_seq_len)
    torch.cuda.synchronize()
    assert torch.equal(base.view(torch.int16), out.view(torch.int16))


def test_shared_pages_across_requests():
    """The same physical pages in two rows (read-only sharing, reading c10)."""
    import torch
    case = Case([300, 300], 32, 8, seed=13)
    bt = case.bt_dev.clone()
    bt[1] = bt[0]
    from paper_2411_01142_b200 import neo
    q = case.q_dev.clone()
    q[1] = q[0]
    out = neo.decode_attn(q, case.k_dev, case.v_dev, bt, case.sl_dev, case.max_seq_len, chunk_tokens=64)
    torch.cuda.synchronize()
    assert torch.equal(out[0].view(torch.int16), out[1].view(torch.int16))


def test_determinism_run_to_run():
    import torch
    case = Case(list(range(1, 2000, 97)), 64, 8, seed=14)
    outs = [case.run(chunk_tokens=64).clone() for _ in range(3)]
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))


def test_empty_context_zero_row():
    import torch
    case = Case([0, 5, 0, 300], 32, 8, seed=15)
    out = case.run(chunk_tokens=64)
    got = case.out_f64(out)
    assert (got[0] == 0).all() and (got[2] == 0).all()
    for b in (1, 3):
        assert within_tol(got[b], case.oracle(b))[0]


def test_workspace_reuse_across_shapes():
    """One workspace, many calls with different shapes: counters stay consistent."""
    from paper_2411_01142_b200 import neo
    ws = neo.make_workspace(64, 64, 8, 4096, chunk_tokens=16)
    for seed, ctx in enumerate([[1000, 2000], [4096], [17, 33, 64], list(range(5, 900, 37))]):
        case = Case(ctx, 32, 8, seed=40 + seed)
        out = case.run(chunk_tokens=16, workspace=ws)
        got = case.out_f64(out)
        for b in range(case.B):
            assert within_tol(got[b], case.oracle(b))[0]


def test_debug_validate_rejects_bad_metadata(monkeypatch):
    import torch
    from paper_2411_01142_b200 import neo
    monkeypatch.setenv("NEO_DEBUG_VALIDATE", "1")
    case = Case([20, 50], 32, 8, seed=16)
    case.run()                                         # valid metadata passes
    bt = case.bt_dev.clone()
    bt[1, 1] = case.npages + 5
    with pytest.raises(neo.NeoError) as e:
        neo.decode_attn(case.q_dev, case.k_dev, case.v_dev, bt, case.sl_dev, case.max_seq_len)
    assert e.value.status == neo.NEO_ERR_INVALID_ARG
    sl = case.sl_dev.clone()
    sl[0] = case.max_seq_len + 1
    with pytest.raises(neo.NeoError):
        neo.decode_attn(case.q_dev, case.k_dev, case.v_dev, case.bt_dev, sl, case.max_seq_len)


@pytest.mark.parametrize("P", [16, 32])
def test_kv_append_then_attend(P):
    """neo_kv_append (P:109-110 read-and-append): poison the new token's slot,
    append its K/V, check the bits landed, then attend over the grown context."""
    import torch
    from paper_2411_01142_b200 import neo
    ctx_new = [1, 16, 17, 33, 200, 512]                    # contexts INCLUDING the new token
    case = Case(ctx_new, 32, 8, P=P, seed=31 + P)
    k_new = np.stack([case.k_req[b][n - 1] for b, n in enumerate(ctx_new)])   # [B][Hkv][D]
    v_new = np.stack([case.v_req[b][n - 1] for b, n in enumerate(ctx_new)])
    for b, n in enumerate(ctx_new):                         # poison the slot the append will fill
        t = n - 1
        case.k_dev[case.table[b, t // P], :, t % P] = float("nan")
        case.v_dev[case.table[b, t // P], :, t % P] = float("nan")
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    neo.kv_append(case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, kn, vn)
    torch.cuda.synchronize()
    for b, n in enumerate(ctx_new):
        t = n - 1
        got = case.k_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy()
        assert np.array_equal(got.view(np.uint16), k_new[b])
        got = case.v_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy()
        assert np.array_equal(got.view(np.uint16), v_new[b])
    check_case(case, 64, f"append P={P}")


@pytest.mark.parametrize("C", [64, -1, -4])
def test_cuda_graph_capture_matches_eager(C):
    """decode_attn launches (PDL attribute, fused combine counters; split and
    grouped kernels) captured in a CUDA graph and replayed give the eager results
    bit for bit, replay after replay."""
    import torch
    from paper_2411_01142_b200 import neo
    cases = [Case([5, 300, 1100, 40, 5000], 32, 8, seed=60 + i) for i in range(3)]
    ws = neo.make_workspace(5, 32, 8, 5000, chunk_tokens=C)
    eager = [c.run(chunk_tokens=C, workspace=ws).clone() for c in cases]
    outs = [torch.empty_like(e) for e in eager]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):                                  # warm-up on the capture stream
        for c, o in zip(cases, outs):
            neo.decode_attn(c.q_dev, c.k_dev, c.v_dev, c.bt_dev, c.sl_dev, c.max_seq_len, out=o, chunk_tokens=C,
                            workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for c, o in zip(cases, outs):
            neo.decode_attn(c.q_dev, c.k_dev, c.v_dev, c.bt_dev, c.sl_dev, c.max_seq_len, out=o, chunk_tokens=C,
                            workspace=ws)
    for rep in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for e, o in zip(eager, outs):
            assert torch.equal(e.view(torch.int16), o.view(torch.int16)), rep


def test_rope_append_then_attend():
    """neo_rope_append: q rotated in place and k rotated into its page slot match the
    fp64 RoPE oracle (tolerance rule), v lands bit-exact, and attention over the
    grown cache matches the oracle on the oracle's rotated inputs."""
    import torch
    from oracle import rope as orope
    import oracle
    from paper_2411_01142_b200 import neo
    ctx_new = [1, 17, 300, 4096]
    case = Case(ctx_new, 32, 8, seed=71)
    P = case.P
    f = orope.llama_inv_freq()
    inv = torch.from_numpy(f).cuda()
    k_new = np.stack([case.k_req[b][n - 1] for b, n in enumerate(ctx_new)])
    v_new = np.stack([case.v_req[b][n - 1] for b, n in enumerate(ctx_new)])
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    q = case.q_dev.clone()
    neo.rope_append(q, inv, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, kn, vn)
    torch.cuda.synchronize()
    q_got = ni.bf16_bits_to_f64(q.view(torch.int16).cpu().numpy().view(np.uint16))
    for b, n in enumerate(ctx_new):
        t = n - 1
        ref_q = orope.rope(ni.bf16_bits_to_f64(case.q[b]), t, f)
        assert within_tol(q_got[b], ref_q)[0]
        k_pg = case.k_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        ref_k = orope.rope(ni.bf16_bits_to_f64(k_new[b]), t, f)
        assert within_tol(ni.bf16_bits_to_f64(k_pg), ref_k)[0]
        v_pg = case.v_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(v_pg, v_new[b])
    out = neo.decode_attn(q, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.max_seq_len)
    torch.cuda.synchronize()
    got = case.out_f64(out)
    for b, n in enumerate(ctx_new):
        t = n - 1
        qr = ni.f32_to_bf16_bits(orope.rope(ni.bf16_bits_to_f64(case.q[b]), t, f).astype(np.float32))
        kr = case.k_req[b].copy()
        kr[t] = ni.f32_to_bf16_bits(orope.rope(ni.bf16_bits_to_f64(k_new[b]), t, f).astype(np.float32))
        ref = oracle.decode_attention(qr, kr, case.v_req[b], np.float32(case.scale))
        assert within_tol(got[b], ref)[0]


@pytest.mark.parametrize("chunk", [0, 64, -1, -4])
def test_decode_attn_append_plain_equals_separate(chunk):
    """neo_decode_attn_append without RoPE == neo_kv_append + neo_decode_attn, bit
    for bit (output and the appended page slots), the new slots poisoned first."""
    import torch
    from paper_2411_01142_b200 import neo
    ctx_new = [1, 16, 17, 300, 1025, 2048, 4097, 5000]
    a = Case(ctx_new, 32, 8, seed=81)
    b = Case(ctx_new, 32, 8, seed=81)
    k_new = np.stack([a.k_req[i][n - 1] for i, n in enumerate(ctx_new)])
    v_new = np.stack([a.v_req[i][n - 1] for i, n in enumerate(ctx_new)])
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    for c in (a, b):
        for i, n in enumerate(ctx_new):
            t = n - 1
            c.k_dev[c.table[i, t // c.P], :, t % c.P] = float("nan")
            c.v_dev[c.table[i, t // c.P], :, t % c.P] = float("nan")
    neo.kv_append(a.k_dev, a.v_dev, a.bt_dev, a.sl_dev, kn, vn)
    ref = a.run(chunk_tokens=chunk)
    got = neo.decode_attn_append(b.q_dev, b.k_dev, b.v_dev, b.bt_dev, b.sl_dev, b.max_seq_len, kn, vn,
                                 chunk_tokens=chunk, scale=b.scale)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))
    for i, n in enumerate(ctx_new):
        t = n - 1
        for pa, pb in ((a.k_dev, b.k_dev), (a.v_dev, b.v_dev)):
            assert torch.equal(pa[a.table[i, t // a.P], :, t % a.P].view(torch.int16),
                               pb[b.table[i, t // b.P], :, t % b.P].view(torch.int16))


@pytest.mark.parametrize("chunk,P", [(0, 16), (64, 16), (0, 32), (-1, 16), (-1, 32)])
def test_decode_attn_append_rope_vs_oracle(chunk, P):
    """The one-launch decode step with RoPE: output within tolerance of the oracle
    over the fp64-rotated q and k (bf16-rounded), the page slot's k within
    tolerance of the rotated k_new, v bit-exact."""
    import torch
    from oracle import rope as orope
    import oracle
    from paper_2411_01142_b200 import neo
    ctx_new = [1, 17, 300, 4096, 700, 4097, 6000]
    case = Case(ctx_new, 32, 8, P=P, seed=91 + P)
    f = orope.llama_inv_freq()
    k_new = np.stack([case.k_req[b][n - 1] for b, n in enumerate(ctx_new)])
    v_new = np.stack([case.v_req[b][n - 1] for b, n in enumerate(ctx_new)])
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    q_before = case.q_dev.clone()
    out = neo.decode_attn_append(case.q_dev, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.max_seq_len, kn,
                                 vn, inv_freq=torch.from_numpy(f).cuda(), chunk_tokens=chunk)
    torch.cuda.synchronize()
    assert torch.equal(case.q_dev.view(torch.int16), q_before.view(torch.int16))     # q not written back
    got = case.out_f64(out)
    for b, n in enumerate(ctx_new):
        t = n - 1
        kr = ni.f32_to_bf16_bits(orope.rope(ni.bf16_bits_to_f64(k_new[b]), t, f).astype(np.float32))
        k_pg = case.k_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        assert within_tol(ni.bf16_bits_to_f64(k_pg), ni.bf16_bits_to_f64(kr))[0]
        v_pg = case.v_dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(v_pg, v_new[b])
        qr = ni.f32_to_bf16_bits(orope.rope(ni.bf16_bits_to_f64(case.q[b]), t, f).astype(np.float32))
        kreq = case.k_req[b].copy()
        kreq[t] = kr
        ref = oracle.decode_attention(qr, kreq, case.v_req[b], np.float32(case.scale))
        ok, ratio = within_tol(got[b], ref)
        assert ok, (b, n, ratio)


# ---- grouped split-K kernel (chunk_tokens = NEO_CHUNK_GROUPED = -1)

GROUPED = -1


@pytest.mark.parametrize("k", [-1, -2, -4, -64, -400, -1536, -3072, -4096])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (64, 8), (32, 32), (28, 4), (24, 8), (8, 1), (40, 8)])
def test_parity_grouped(hq, hkv, k):
    """One CTA per group of <= 256 / -k tiles, 4 per-warp ranges merged in shared
    memory; longer requests run several groups and the cross-group combine."""
    ctx = [1, 15, 16, 17, 63, 65, 255, 256, 257, 1000, 1025, 2049, 4095, 4096, 4097, 4111, 8192, 9000]
    check_case(Case(ctx, hq, hkv, seed=21 + hq + hkv), k, f"grouped{k} G={hq // hkv}")


@pytest.mark.parametrize("k", [-1, -4])
@pytest.mark.parametrize("P", [32, 64])
def test_parity_grouped_page_sizes(P, k):
    check_case(Case([1, 31, 32, 33, 700, 1100, 5000], 32, 8, P=P, seed=22 + P), k, f"grouped{k} P={P}")


@pytest.mark.parametrize("variant", [ni.VARIANT_PEAKED, ni.VARIANT_SINK, ni.VARIANT_PEAKED | ni.VARIANT_SINK])
def test_parity_grouped_variants(variant):
    check_case(Case([3, 500, 1100, 4500], 64, 8, seed=23, variant=variant), GROUPED, f"grouped variant={variant}")


def test_grouped_empty_determinism_and_batch_independence():
    """Empty contexts give zero rows; outputs are bitwise run to run and a request's
    row does not depend on the other requests of the batch (the split is a function
    of its own length)."""
    import torch
    full = Case([0, 5, 0, 300, 4200, 1000], 32, 8, seed=24)
    outs = [full.run(chunk_tokens=GROUPED).clone() for _ in range(3)]
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))
    got = full.out_f64(outs[0])
    assert (got[0] == 0).all() and (got[2] == 0).all()
    for b in (1, 3, 4, 5):
        assert within_tol(got[b], full.oracle(b))[0]


def test_grouped_workspace_reuse():
    """The multi-group combine leaves its counters at zero: a reused workspace
    gives bitwise the same output (graph capture: test_cuda_graph_capture_matches_eager)."""
    import torch

    from paper_2411_01142_b200 import neo
    case = Case([100, 4500, 9000, 33], 32, 8, seed=25)
    ws = neo.make_workspace(case.B, 32, 8, case.max_seq_len, GROUPED)
    eager = case.run(chunk_tokens=GROUPED, workspace=ws).clone()
    again = case.run(chunk_tokens=GROUPED, workspace=ws).clone()
    assert torch.equal(eager.view(torch.int16), again.view(torch.int16))


# ---- NEO_ATTN_KV_STABLE (neo_decode_attn_ex): metadata and first KV tiles before the PDL wait


@pytest.mark.parametrize("chunk", [0, 64, 640, -1, -2, -1536])
def test_kv_stable_after_append_is_bitwise_and_sees_new_token(chunk):
    """A PDL neo_kv_append of every request's newest token immediately followed
    by a kv_stable attention call (its first KV tiles read before the wait): the
    newest token's tile is never read early, so the output is bitwise the output
    of the plain call and within tolerance of the oracle -- repeated, with the
    newest slots re-poisoned with NaN before every append."""
    import torch
    from paper_2411_01142_b200 import neo
    ctx_new = [1, 2, 16, 17, 33, 64, 65, 200, 512, 1000, 2049, 4100]
    case = Case(ctx_new, 32, 8, seed=91)
    P = case.P
    k_new = np.stack([case.k_req[b][n - 1] for b, n in enumerate(ctx_new)])
    v_new = np.stack([case.v_req[b][n - 1] for b, n in enumerate(ctx_new)])
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    ws = neo.make_workspace(case.B, 32, 8, case.max_seq_len, chunk)
    ref = neo.decode_attn(case.q_dev, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.max_seq_len,
                          chunk_tokens=chunk, workspace=ws).clone()
    got = case.out_f64(ref)
    for b in range(case.B):
        assert within_tol(got[b], case.oracle(b))[0]
    pages = torch.tensor([int(case.table[b, (n - 1) // P]) for b, n in enumerate(ctx_new)], device="cuda")
    slots = torch.tensor([(n - 1) % P for n in ctx_new], device="cuda")
    out = torch.empty_like(ref)
    for rep in range(12):
        case.k_dev[pages, :, slots] = float("nan")
        case.v_dev[pages, :, slots] = float("nan")
        neo.kv_append(case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, kn, vn)
        neo.decode_attn(case.q_dev, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.max_seq_len, out=out,
                        chunk_tokens=chunk, workspace=ws, kv_stable=True)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16)), rep


@pytest.mark.parametrize("chunk", [512, -1, -2])
def test_kv_stable_back_to_back_layers(chunk):
    """Three layer pools called back to back with kv_stable (the bench's decode
    step): every output bitwise equals its plain call."""
    import torch
    from paper_2411_01142_b200 import neo
    cases = [Case([5, 300, 1100, 40, 5000, 2048], 64, 8, seed=95 + i, layer=i) for i in range(3)]
    ws = neo.make_workspace(6, 64, 8, 5000, chunk_tokens=chunk)
    plain = [c.run(chunk_tokens=chunk, workspace=ws).clone() for c in cases]
    outs = [torch.empty_like(p) for p in plain]
    for rep in range(5):
        for c, o in zip(cases, outs):
            neo.decode_attn(c.q_dev, c.k_dev, c.v_dev, c.bt_dev, c.sl_dev, c.max_seq_len, out=o, chunk_tokens=chunk,
                            workspace=ws, kv_stable=True)
        torch.cuda.synchronize()
        for p, o in zip(plain, outs):
            assert torch.equal(p.view(torch.int16), o.view(torch.int16)), rep


def test_kv_stable_rejects_unknown_flags():
    import torch
    from paper_2411_01142_b200 import neo
    c = Case([10, 20], 32, 8, seed=97)
    ws = neo.make_workspace(2, 32, 8, c.max_seq_len, 64)
    out = torch.empty_like(c.q_dev)
    rc = neo.lib().neo_decode_attn_ex(c.q_dev.data_ptr(), c.k_dev.data_ptr(), c.v_dev.data_ptr(), c.k_dev.stride(0),
                                      c.k_dev.shape[0], c.bt_dev.data_ptr(), c.bt_dev.shape[1], c.sl_dev.data_ptr(),
                                      out.data_ptr(), 2, 32, 8, 128, 16, c.max_seq_len, 0.088, 64, ws.data_ptr(),
                                      ws.numel(), 2, None)
    assert rc == neo.NEO_ERR_INVALID_ARG
