"""GPU parity of the prefill side of batch-0 through
the C ABI: neo_prefill_append (ragged multi-token KV store, optional RoPE)
against the fp64 RoPE oracle / bit copies, and neo_prefill_attn against the
fp64 causal prefill oracle under the north-star tolerance rule."""
import numpy as np
import pytest

import neo_inputs as ni
from harness import PrefillCase, within_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def _page_row(dev, case, b, t):
    P = case.P
    import torch
    return dev[case.table[b, t // P], :, t % P].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("rope", [False, True])
def test_prefill_append(rope):
    import torch
    from oracle import rope as orope
    from paper_2411_01142_b200 import neo
    ctx = [1, 40, 300, 129, 1000, 17]
    q_lens = [1, 40, 100, 1, 1000, 0]          # whole prompts, a chunk after a prefix, single tokens, empty
    case = PrefillCase(ctx, q_lens, 32, 8, seed=91 + rope)
    f = orope.llama_inv_freq()
    k_new = np.concatenate([case.k_req[b][n - m:] for b, (n, m) in enumerate(zip(ctx, q_lens))])
    v_new = np.concatenate([case.v_req[b][n - m:] for b, (n, m) in enumerate(zip(ctx, q_lens))])
    for b, (n, m) in enumerate(zip(ctx, q_lens)):              # poison the slots the store fills
        for t in range(n - m, n):
            case.k_dev[case.table[b, t // case.P], :, t % case.P] = float("nan")
            case.v_dev[case.table[b, t // case.P], :, t % case.P] = float("nan")
    kn = torch.from_numpy(k_new.view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(v_new.view(np.int16)).cuda().view(torch.bfloat16)
    q = case.qp_dev.clone()
    neo.prefill_append(case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.qo_dev, kn, vn,
                       q=q if rope else None, inv_freq=torch.from_numpy(f).cuda() if rope else None)
    torch.cuda.synchronize()
    q_got = q.view(torch.int16).cpu().numpy().view(np.uint16)
    if not rope:
        assert np.array_equal(q_got, case.qp)
    for b, (n, m) in enumerate(zip(ctx, q_lens)):
        for i, t in enumerate(range(n - m, n)):
            j = case.q_off[b] + i
            assert np.array_equal(_page_row(case.v_dev, case, b, t), case.v_req[b][t])
            kg = _page_row(case.k_dev, case, b, t)
            if not rope:
                assert np.array_equal(kg, case.k_req[b][t])
                continue
            assert within_tol(ni.bf16_bits_to_f64(kg), orope.rope(ni.bf16_bits_to_f64(case.k_req[b][t]), t, f))[0]
            assert within_tol(ni.bf16_bits_to_f64(q_got[j]), orope.rope(ni.bf16_bits_to_f64(case.qp[j]), t, f))[0]


def check_prefill(case, tag=""):
    out = case.run()
    got = ni.bf16_bits_to_f64(out.view(__import__("torch").int16).cpu().numpy().view(np.uint16))
    worst = 0.0
    for b in range(case.B):
        if case.q_lens[b] == 0:
            continue
        ok, ratio = within_tol(got[case.rows(b)], case.oracle(b))
        worst = max(worst, ratio)
        assert ok, f"{tag} b={b} ctx={case.ctx[b]} q_len={case.q_lens[b]} err/tol={ratio:.3f}"
    return out, worst


@pytest.mark.parametrize("hq,hkv", [(32, 8), (8, 8), (16, 8), (64, 8), (16, 1)])
def test_prefill_parity_whole_prompts(hq, hkv):
    ctx = [1, 7, 64, 65, 128, 300, 1000]
    check_prefill(PrefillCase(ctx, ctx, hq, hkv, seed=100 + hq + hkv), f"hq={hq} hkv={hkv}")


@pytest.mark.parametrize("P", [16, 32, 64])
def test_prefill_parity_chunks_after_prefix(P):
    ctx = [500, 200, 129, 64, 1500, 33]
    q_lens = [100, 1, 64, 0, 257, 33]        # chunked prefill after a cached prefix, a single token, an empty slot
    check_prefill(PrefillCase(ctx, q_lens, 32, 8, P=P, seed=200 + P), f"P={P}")


@pytest.mark.parametrize("variant", [1, 2])
def test_prefill_parity_variants(variant):
    ctx = [700, 96, 1200]
    check_prefill(PrefillCase(ctx, [700, 50, 300], 32, 8, variant=variant, seed=300 + variant), f"variant={variant}")


def test_prefill_determinism_and_nan_tails():
    import torch
    ctx = [77, 1000, 513]
    case = PrefillCase(ctx, ctx, 32, 8, seed=400)            # page tails are NaN-poisoned by the harness
    a = case.run().clone()
    b = case.run()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.isfinite(a.float()).all()


def test_prefill_last_row_matches_decode():
    """The last prompt row at position n-1 is exactly a decode query over all n tokens:
    prefill and decode kernels agree within the tolerance on it."""
    import torch
    from paper_2411_01142_b200 import neo
    ctx = [300, 1024, 77]
    case = PrefillCase(ctx, ctx, 32, 8, seed=500)
    out = case.run()
    last = torch.stack([case.qp_dev[case.q_off[b + 1] - 1] for b in range(case.B)]).contiguous()
    dec = neo.decode_attn(last, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.max_seq_len)
    torch.cuda.synchronize()
    for b in range(case.B):
        a = ni.bf16_bits_to_f64(out[case.q_off[b + 1] - 1].view(torch.int16).cpu().numpy().view(np.uint16))
        d = ni.bf16_bits_to_f64(dec[b].view(torch.int16).cpu().numpy().view(np.uint16))
        assert within_tol(a, d)[0]


def test_prefill_parity_many_ragged_requests():
    """40 requests of random prompt / prefix lengths (some empty): the dense
    longest-first schedule table covers every (request, kv-head, tile) once."""
    rng = np.random.default_rng(600)
    ctx = rng.integers(1, 400, 40)
    q_lens = np.minimum(ctx, rng.integers(0, 300, 40))
    q_lens[::7] = 0
    check_prefill(PrefillCase(ctx.tolist(), q_lens.tolist(), 32, 8, seed=601), "ragged40")


def test_prefill_cuda_graph_matches_eager():
    """neo_prefill_append (RoPE) + neo_prefill_attn -- PDL launches, persistent
    grid -- captured in a CUDA graph and replayed give the eager bits."""
    import torch
    from oracle import rope as orope
    from paper_2411_01142_b200 import neo
    ctx = [300, 77, 1000]
    case = PrefillCase(ctx, [300, 40, 1000], 32, 8, seed=700)
    inv = torch.from_numpy(orope.llama_inv_freq()).cuda()
    kn = torch.zeros(case.T, 8, 128, dtype=torch.bfloat16, device="cuda").normal_(generator=torch.Generator("cuda").manual_seed(1))
    vn = torch.zeros_like(kn).normal_(generator=torch.Generator("cuda").manual_seed(2))
    q = case.qp_dev.clone()
    out = torch.empty_like(q)

    def step(stream=None):
        q.copy_(case.qp_dev)
        neo.prefill_append(case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.qo_dev, kn, vn, q=q, inv_freq=inv,
                           stream=stream)
        neo.prefill_attn(q, case.k_dev, case.v_dev, case.bt_dev, case.sl_dev, case.qo_dev, case.max_q_len, out=out,
                         stream=stream)

    step()
    torch.cuda.synchronize()
    eager = out.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream())
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), eager.view(torch.int16))


@pytest.mark.parametrize("n,variant", [(8192, 0), (16384, 0), (8192, ni.VARIANT_PEAKED),
                                       (16384, ni.VARIANT_PEAKED), (16384, ni.VARIANT_PEAKED | ni.VARIANT_SINK),
                                       (8192, ni.VARIANT_SINK)])
def test_prefill_parity_long_prompts_sampled(n, variant):
    """Whole 8K / 16K prompts (the lengths DESIGN §11 quotes TF/s for), plain,
    peaked (q x 8: the running max keeps growing, so the lazy O rescale -- only
    when the max grows by > 2^8 -- fires with P up to 2^8 accumulated) and
    attention-sink inputs.  The oracle checks sampled rows one by one: each row
    is the decode definition over its visible prefix (tile edges, page edges,
    the first and last rows, and random rows)."""
    import os
    import oracle
    import torch
    case = PrefillCase([n], [n], 32, 8, seed=800 + n // 1024 + variant, variant=variant)
    out = case.run()
    got = ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))
    rng = np.random.default_rng(n + variant)
    rows = sorted(set([0, 1, 15, 16, 17, 127, 128, 129, 255, 256, 1000, 4095, 4096, n // 2, n - 129, n - 128,
                       n - 2, n - 1] + rng.integers(0, n, 30).tolist()))
    q = case.qp[rows]
    ks = [case.k_req[0][:i + 1] for i in rows]
    vs = [case.v_req[0][:i + 1] for i in rows]
    ref = oracle.decode_attention_batch(q, ks, vs, np.float32(case.scale), nthreads=os.cpu_count() or 1)
    worst = 0.0
    for j, i in enumerate(rows):
        ok, ratio = within_tol(got[i], ref[j])
        worst = max(worst, ratio)
        assert ok, f"n={n} variant={variant} row={i} err/tol={ratio:.3f}"


@pytest.mark.parametrize("kernel", ["item", "stream"])
def test_prefill_long_prompt_both_fp16_kernels(kernel, monkeypatch):
    """An 8K whole prompt with peaked logits (the lazy O rescale fires) through
    both fp16 kernels: the launch picks the item-major one at this length, the
    stream kernel (NEO_PREFILL_KERNEL=stream) must be exact at any length too."""
    import os
    import oracle
    import torch
    monkeypatch.setenv("NEO_PREFILL_KERNEL", kernel)
    n = 8192
    case = PrefillCase([n], [n], 32, 8, seed=850, variant=ni.VARIANT_PEAKED)
    out = case.run()
    got = ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))
    rng = np.random.default_rng(851)
    rows = sorted(set([0, 31, 32, 63, 64, 127, 128, 4095, 4096, n - 65, n - 64, n - 1] + rng.integers(0, n, 20).tolist()))
    ref = oracle.decode_attention_batch(case.qp[rows], [case.k_req[0][:i + 1] for i in rows],
                                        [case.v_req[0][:i + 1] for i in rows], np.float32(case.scale),
                                        nthreads=os.cpu_count() or 1)
    for j, i in enumerate(rows):
        ok, ratio = within_tol(got[i], ref[j])
        assert ok, f"{kernel} row={i} err/tol={ratio:.3f}"


@pytest.mark.parametrize("pv,kernel", [("hilo", "item"), ("fp16", "item"), ("fp16", "stream")])
def test_prefill_both_pv_paths(pv, kernel, monkeypatch):
    """Every prefill kernel variant (DESIGN "prefill P.V": fp16 P with V converted
    to fp16 in shared memory -- item-major or stream kernel -- or the bf16 hi + lo
    split; the launch picks by prompt length, NEO_PREFILL_PV / NEO_PREFILL_KERNEL
    force one) on short and long prompts, chunks after a prefix, single-tile items
    and page-size 32 pools, against the oracle."""
    monkeypatch.setenv("NEO_PREFILL_PV", pv)
    monkeypatch.setenv("NEO_PREFILL_KERNEL", kernel)
    check_prefill(PrefillCase([1, 7, 64, 65, 128, 300, 1000], [1, 7, 64, 65, 128, 300, 1000], 64, 8,
                              seed=900), f"{pv} G=8")
    check_prefill(PrefillCase([500, 200, 129, 1500, 33], [100, 1, 64, 257, 33], 32, 8, P=32, seed=901),
                  f"{pv} P=32")
    check_prefill(PrefillCase([77, 2100], [77, 2100], 16, 1, seed=902, variant=ni.VARIANT_PEAKED), f"{pv} G=16")


def test_prefill_slow_epilogue_one_step_items():
    """Barrier-phase regression (stream kernel): with the epilogue slowed down
    (NEO_PREFILL_EPI_DELAY_NS sleeps before each item's epilogue), the softmax
    warps of a CTA working through one-step items would complete l_ready twice
    before the epilogue waits on it and alias its parity -- a hang -- unless
    they wait o_free of the previous item first.  Run in a subprocess with a
    timeout, so a regression fails the test instead of hanging the suite."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    ctx = ",".join(["300"] + ["64"] * 60 + ["1", "17"])
    env = dict(os.environ, NEO_PREFILL_KERNEL="stream", NEO_PREFILL_EPI_DELAY_NS="200000")
    try:
        r = subprocess.run([sys.executable, os.path.join(here, "_prefill_slow_epilogue.py"), ctx], env=env,
                           capture_output=True, text=True, timeout=180)
    except subprocess.TimeoutExpired:
        pytest.fail("stream prefill kernel hung with a slow epilogue (l_ready parity aliasing)")
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_prefill_stream_item_list_overflow(monkeypatch):
    """The stream kernel decodes at most 512 items per CTA into shared memory in
    its prologue and decodes later ones on the fly: a grid capped to 2 CTAs
    (NEO_PREFILL_CTAS, the SM-budget knob) over 1152 items runs 576 rounds per
    CTA, so the on-the-fly path is exercised; parity against the oracle."""
    monkeypatch.setenv("NEO_PREFILL_KERNEL", "stream")
    monkeypatch.setenv("NEO_PREFILL_CTAS", "2")
    ctx = [1000] * 9
    check_prefill(PrefillCase(ctx, ctx, 32, 8, seed=960), "stream, 2 CTAs, 576 rounds each")
