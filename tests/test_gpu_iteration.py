"""NEO iterations end to end through the C ABI (SURVEY §8(f) rows working
together), on an attention-only toy model of L layers.

Every iteration:
1. `neo_schedule` plans batch-0 / batch-1 and the swaps from a toy cost profile and the pool's free pages.
2. `neo_kv_swap_out` / `neo_kv_swap_in` move whole requests between the GPU-cache and the CPU-cache.
3. Admitted prompts are prefilled on the GPU with `neo_prefill_append` (RoPE) and `neo_prefill_attn`.
4. GPU-resident requests decode one token with the one-launch `neo_decode_attn_append` (RoPE + append + attention).
5. CPU-resident requests decode with `neo_cpu_decode_attn` over the CPU-cache pages.

Every attention output is checked against the fp64 oracle over the request's
full K/V history, under the north-star tolerance.  Per-token q / k / v come from
the seeded counter-based generator (no model weights); the RoPE the test
applies to the CPU requests' q / k (NEO computes them on the GPU) is the
oracle's (test infrastructure)."""
import math

import numpy as np
import pytest

import neo_inputs as ni
from harness import within_tol

pytestmark = pytest.mark.gpu

L, HQ, HKV, D, P = 2, 32, 8, 128, 16
SEED = 0x4E454F


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def _qkv(layer, rid, pos):
    """q [n][Hq][D], k / v [n][Hkv][D] bf16 bits of request rid's tokens `pos`."""
    ids = np.asarray(pos, dtype=np.int64) + 100000 * rid
    return (ni.q_bits(SEED, 1000 + layer, ids, HQ, D), ni.q_bits(SEED, 2000 + layer, ids, HKV, D),
            ni.q_bits(SEED, 3000 + layer, ids, HKV, D))


TOY_PROFILE = {
    "L": L, "t_prl": 1e-5, "t_pol": 1e-5,
    "lin": [[1, 1e-6], [8192, 8e-3]],              # linear stage ~ proportional to tokens
    "gdec": [[1, 1e-6], [1 << 20, 1e-3]],
    "gpre_a": 1e-12, "gpre_b": 1e-8,
    "cdec": [[1, 1e-7], [1 << 20, 1e-4]],          # cheap CPU attention: two-batch plans pay
    "page_size": P, "max_batch_tokens": 512, "pcie_bytes_per_s": 50e9,
    "kv_bytes_per_token_layer": HKV * D * 2 * 2,
}


def test_neo_iterations_end_to_end():
    import torch
    from oracle import rope as orope
    import oracle
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo

    prompts = [50, 120, 33, 90, 64, 40]
    outputs = [12, 10, 16, 9, 14, 11]
    GPU_PAGES, HOST_PAGES = 14, 120                # the prompts alone need 28 pages: the GPU-cache overflows
    pool = neo.KVPool(L, HKV, num_gpu_pages=GPU_PAGES, num_host_pages=HOST_PAGES, page_size=P)
    gpu_free = lambda: pool.free_count(NEO_GPU)    # noqa: E731
    cpu_free = lambda: pool.free_count(NEO_HOST)   # noqa: E731
    f = orope.llama_inv_freq()
    inv = torch.from_numpy(f).cuda()
    scale = 1 / math.sqrt(D)
    staging = torch.empty(pool.staging_bytes(16), dtype=torch.uint8, device="cuda")
    R = len(prompts)
    st = [{"where": "wait", "ctx": 0, "gen": 0, "gpu": [], "host": []} for _ in range(R)]
    hist_k = [[np.zeros((0, HKV, D), np.uint16) for _ in range(L)] for _ in range(R)]   # rotated K bits
    hist_v = [[np.zeros((0, HKV, D), np.uint16) for _ in range(L)] for _ in range(R)]
    rot = lambda bits, pos: ni.f32_to_bf16_bits(np.stack(  # noqa: E731
        [orope.rope(ni.bf16_bits_to_f64(bits[i]), int(p), f) for i, p in enumerate(pos)]).astype(np.float32))
    to_dev = lambda bits: torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)  # noqa
    bits = lambda t: t.view(torch.int16).cpu().numpy().view(np.uint16)   # noqa: E731
    counts = {"prefill": 0, "gpu_decode": 0, "cpu_decode": 0, "swap_out": 0, "swap_in": 0, "two_batch": 0}

    def table(rids, key, width):
        t = np.zeros((max(len(rids), 1), width), dtype=np.int32)
        for i, r in enumerate(rids):
            t[i, :len(st[r][key])] = st[r][key]
        return t

    def grow_pages(r, where):
        key = "gpu" if where == NEO_GPU else "host"
        while len(st[r][key]) * P < st[r]["ctx"] + 1:
            st[r][key] += pool.alloc(where, 1).tolist()

    def swap(r, out_dir):
        n = len(st[r]["gpu" if out_dir else "host"])
        if out_dir:
            host = pool.alloc(NEO_HOST, n)
            pool.swap_out(st[r]["gpu"], host, staging)
            torch.cuda.synchronize()
            pool.free(NEO_GPU, st[r]["gpu"])
            st[r]["gpu"], st[r]["host"], st[r]["where"] = [], host.tolist(), "cpu"
        else:
            gids = pool.alloc(NEO_GPU, n)
            pool.swap_in(st[r]["host"], gids, staging)
            torch.cuda.synchronize()
            pool.free(NEO_HOST, st[r]["host"])
            st[r]["gpu"], st[r]["host"], st[r]["where"] = gids.tolist(), [], "gpu"

    for _ in range(200):
        live = [r for r in range(R) if st[r]["where"] != "done"]
        if not live:
            break
        kinds = {"wait": 0, "gpu": 1, "cpu": 2}
        order = [(r, kinds[st[r]["where"]], st[r]["ctx"] if st[r]["where"] != "wait" else prompts[r])
                 for w in ("gpu", "wait", "cpu") for r in live if st[r]["where"] == w]
        plan = neo.schedule(TOY_PROFILE, order, gpu_free(), cpu_free())
        counts["two_batch"] += plan["two_batch"]
        for r in plan["swap_in"]:
            swap(r, False)
            counts["swap_in"] += 1
        pre_out = set()
        for r in plan["swap_out"]:
            if st[r]["where"] == "gpu":
                swap(r, True)
                counts["swap_out"] += 1
            else:
                pre_out.add(r)                       # prefill whose KV goes to the CPU-cache
        batch = plan["batch0"] + plan["batch1"]
        if not batch:
            continue

        # ---- prefill (batch-0 prompts) on the GPU
        pre = [r for r in batch if st[r]["where"] == "wait"]
        if pre:
            for r in pre:
                st[r]["gpu"] = pool.alloc(NEO_GPU, -(-prompts[r] // P)).tolist()
            bt = torch.from_numpy(table(pre, "gpu", max(len(st[r]["gpu"]) for r in pre))).cuda()
            sl = torch.tensor([prompts[r] for r in pre], dtype=torch.int32, device="cuda")
            qoff = np.concatenate([[0], np.cumsum([prompts[r] for r in pre])]).astype(np.int32)
            qo = torch.from_numpy(qoff).cuda()
            for layer in range(L):
                qkv = [_qkv(layer, r, np.arange(prompts[r])) for r in pre]
                q = to_dev(np.concatenate([x[0] for x in qkv]))
                kn, vn = to_dev(np.concatenate([x[1] for x in qkv])), to_dev(np.concatenate([x[2] for x in qkv]))
                k_pages, v_pages = pool.layer_view(layer)
                neo.prefill_append(k_pages, v_pages, bt, sl, qo, kn, vn, q=q, inv_freq=inv)
                out = bits(neo.prefill_attn(q, k_pages, v_pages, bt, sl, qo, max(prompts[r] for r in pre)))
                for i, r in enumerate(pre):
                    pos = np.arange(prompts[r])
                    kr, qr = rot(qkv[i][1], pos), rot(qkv[i][0], pos)
                    hist_k[r][layer], hist_v[r][layer] = kr, qkv[i][2]
                    ref = oracle.prefill_attention(qr, kr, qkv[i][2], scale)
                    assert within_tol(ni.bf16_bits_to_f64(out[qoff[i]:qoff[i + 1]]), ref)[0], ("prefill", r, layer)
            for r in pre:
                st[r].update(where="gpu", ctx=prompts[r], gen=1)
                counts["prefill"] += 1
                if r in pre_out:
                    swap(r, True)

        # ---- GPU decode: one token per request, RoPE + append + attention in one launch per layer
        gd = [r for r in batch if st[r]["where"] == "gpu" and r not in pre]
        if gd:
            for r in gd:
                grow_pages(r, NEO_GPU)
            bt = torch.from_numpy(table(gd, "gpu", max(len(st[r]["gpu"]) for r in gd))).cuda()
            sl = torch.tensor([st[r]["ctx"] + 1 for r in gd], dtype=torch.int32, device="cuda")
            for layer in range(L):
                qkv = [_qkv(layer, r, [st[r]["ctx"]]) for r in gd]
                k_pages, v_pages = pool.layer_view(layer)
                out = bits(neo.decode_attn_append(
                    to_dev(np.concatenate([x[0] for x in qkv])), k_pages, v_pages, bt, sl,
                    max(st[r]["ctx"] + 1 for r in gd), to_dev(np.concatenate([x[1] for x in qkv])),
                    to_dev(np.concatenate([x[2] for x in qkv])), inv_freq=inv))
                for i, r in enumerate(gd):
                    t = st[r]["ctx"]
                    hist_k[r][layer] = np.concatenate([hist_k[r][layer], rot(qkv[i][1], [t])])
                    hist_v[r][layer] = np.concatenate([hist_v[r][layer], qkv[i][2]])
                    ref = oracle.decode_attention(rot(qkv[i][0], [t])[0], hist_k[r][layer], hist_v[r][layer], scale)
                    assert within_tol(ni.bf16_bits_to_f64(out[i]), ref)[0], ("gpu decode", r, layer)
            for r in gd:
                st[r]["ctx"] += 1
                st[r]["gen"] += 1
                counts["gpu_decode"] += 1

        # ---- CPU decode (batch-0 and batch-1 CPU-requests): the new token's rotated
        # k / v go into the CPU-cache page (TrQKV), then CPU attention
        cd = [r for r in batch if st[r]["where"] == "cpu" and r not in pre]
        if cd:
            for r in cd:
                grow_pages(r, NEO_HOST)
            ht = table(cd, "host", max(len(st[r]["host"]) for r in cd))
            hv = pool.host_view()
            for layer in range(L):
                qs = []
                for r in cd:
                    t = st[r]["ctx"]
                    q1, k1, v1 = _qkv(layer, r, [t])
                    kr = rot(k1, [t])
                    page = st[r]["host"][t // P]
                    hv[page, layer, 0, :, t % P] = torch.from_numpy(kr[0].view(np.int16)).view(torch.bfloat16)
                    hv[page, layer, 1, :, t % P] = torch.from_numpy(v1[0].view(np.int16)).view(torch.bfloat16)
                    hist_k[r][layer] = np.concatenate([hist_k[r][layer], kr])
                    hist_v[r][layer] = np.concatenate([hist_v[r][layer], v1])
                    qs.append(rot(q1, [t])[0])
                out = pool.cpu_decode_attn(layer, np.stack(qs), ht, [st[r]["ctx"] + 1 for r in cd])
                for i, r in enumerate(cd):
                    ref = oracle.decode_attention(qs[i], hist_k[r][layer], hist_v[r][layer], scale)
                    assert within_tol(ni.bf16_bits_to_f64(out[i]), ref)[0], ("cpu decode", r, layer)
            for r in cd:
                st[r]["ctx"] += 1
                st[r]["gen"] += 1
                counts["cpu_decode"] += 1

        for r in batch:                              # finished requests release their pages
            if st[r]["gen"] >= outputs[r]:
                if st[r]["gpu"]:
                    pool.free(NEO_GPU, st[r]["gpu"])
                if st[r]["host"]:
                    pool.free(NEO_HOST, st[r]["host"])
                st[r].update(where="done", gpu=[], host=[])

    assert all(s["where"] == "done" for s in st), [s["where"] for s in st]
    assert counts["prefill"] == R
    assert counts["gpu_decode"] > 0 and counts["cpu_decode"] > 0, counts
    assert counts["swap_out"] > 0 and counts["swap_in"] > 0 and counts["two_batch"] > 0, counts
    assert pool.free_count(NEO_GPU) == GPU_PAGES and pool.free_count(NEO_HOST) == HOST_PAGES
    print(counts)
