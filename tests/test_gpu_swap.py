"""KV page swap between the GPU-cache and the pinned CPU-cache (P:240,
P:285-288), bit-exact against the oracle's gather definition (SURVEY §8(c)
items 11-13), through the C ABI."""
import numpy as np
import pytest

import oracle
from harness import within_tol

pytestmark = pytest.mark.gpu

SEED = 0x4E454F


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def make_pool(L=4, hkv=8, npages=64, nhost=64, P=16):
    import torch
    from paper_2411_01142_b200 import neo
    pool = neo.KVPool(L, hkv, num_gpu_pages=npages, num_host_pages=nhost, page_size=P)
    g = torch.Generator(device="cuda").manual_seed(1)
    bits = torch.randint(-32768, 32767, (pool.gpu.numel(),), dtype=torch.int16, device="cuda", generator=g)
    pool.gpu.view(torch.int16).copy_(bits)
    pool.host.view(torch.int16).fill_(0x7FC0)
    return pool


def gpu_np(pool):
    import torch
    return pool.gpu_view().view(torch.int16).cpu().numpy().view(np.uint16)


def host_np(pool):
    import torch
    return pool.host_view().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("l0,l1", [(0, 4), (1, 3), (3, 4)])
@pytest.mark.parametrize("staging_pages", [100, 7, 3, 2, 1, 0])
def test_swap_out_matches_gather_definition(l0, l1, staging_pages):
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST
    pool = make_pool()
    gids = pool.alloc(NEO_GPU, 40)
    sel = gids[[5, 17, 2, 33, 8, 9, 10, 11, 39]]
    hids = pool.alloc(NEO_HOST, 12)[[0, 1, 2, 7, 8, 9, 10, 4, 5]]      # several contiguous runs
    staging = (torch.empty(pool.staging_bytes(staging_pages, l0, l1), dtype=torch.uint8, device="cuda")
               if staging_pages else None)                    # 0: zero-copy path
    before = gpu_np(pool)
    pool.swap_out(sel, hids, staging, l0, l1)
    torch.cuda.synchronize()
    rec = oracle.host_record(host_np(pool), hids, l0, l1)
    ref = oracle.gather_pages(before, sel, l0, l1)
    assert np.array_equal(rec, ref)
    # layers outside the range untouched (still the NaN fill)
    untouched = [l for l in range(4) if not (l0 <= l < l1)]
    if untouched:
        assert (host_np(pool)[hids][:, untouched] == 0x7FC0).all()
    assert np.array_equal(gpu_np(pool), before)          # swap-out does not modify the GPU-cache


@pytest.mark.parametrize("zero_copy", [False, True])
def test_swap_in_roundtrip_to_new_ids(zero_copy):
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST
    pool = make_pool()
    old = pool.alloc(NEO_GPU, 10)
    hids = pool.alloc(NEO_HOST, 10)
    staging = None if zero_copy else torch.empty(pool.staging_bytes(4), dtype=torch.uint8, device="cuda")
    before = gpu_np(pool)
    pool.swap_out(old, hids, staging)
    ev = torch.cuda.Event()
    ev.record()
    ev.synchronize()
    pool.free(NEO_GPU, old)
    new = pool.alloc(NEO_GPU, 10)
    # scramble the destination pages first
    pool.gpu_view()[:, :, torch.from_numpy(new.astype(np.int64)).cuda()] = 0
    pool.swap_in(hids, new, staging)
    torch.cuda.synchronize()
    after = gpu_np(pool)
    assert np.array_equal(oracle.gather_pages(after, new, 0, 4), oracle.gather_pages(before, old, 0, 4))


def test_attention_bitwise_after_swap_cycle():
    """Swap a request out and back in to different page ids: attention output is
    bitwise identical (item 13)."""
    import torch
    import neo_inputs as ni
    from neo_inputs import device as gen
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo
    L, hkv, hq, P = 3, 8, 32, 16
    ctx = np.array([333, 1000, 17], dtype=np.int32)
    need = ni.pages_needed(ctx, P)
    pool = neo.KVPool(L, hkv, num_gpu_pages=int(need.sum()) * 2 + 5, num_host_pages=int(need.sum()), page_size=P)
    table = np.full((3, int(need.max())), -1, dtype=np.int32)
    for b in range(3):
        table[b, :need[b]] = pool.alloc(NEO_GPU, int(need[b]))
    bt = torch.from_numpy(table).cuda()
    sl = torch.from_numpy(ctx).cuda()
    q = torch.empty(3, hq, 128, dtype=torch.bfloat16, device="cuda")
    outs = []
    for layer in range(L):
        k, v = pool.layer_view(layer)
        gen.fill_kv(k, v, bt, sl, seed=SEED, layer=layer, hq_total=hq)
    staging = torch.empty(pool.staging_bytes(int(need[1])), dtype=torch.uint8, device="cuda")

    def attn_all(btab):
        res = []
        for layer in range(L):
            gen.fill_q(q, seed=SEED, layer=layer)
            k, v = pool.layer_view(layer)
            res.append(neo.decode_attn(q, k, v, btab, sl, int(ctx.max()), chunk_tokens=64).clone())
        torch.cuda.synchronize()
        return res

    outs = attn_all(bt)
    hids = pool.alloc(NEO_HOST, int(need[1]))
    old = table[1, :need[1]].copy()
    pool.swap_out(old, hids, staging)
    torch.cuda.synchronize()
    pool.free(NEO_GPU, old)
    pool.alloc(NEO_GPU, 3)                                # shift the free list
    new = pool.alloc(NEO_GPU, int(need[1]))
    assert not np.array_equal(new, old)
    pool.swap_in(hids, new, staging)
    table[1, :need[1]] = new
    outs2 = attn_all(torch.from_numpy(table).cuda())
    for a, b in zip(outs, outs2):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    # and the values are right
    import oracle as orc
    for layer in range(L):
        qb = ni.q_bits(SEED, layer, [1], hq, 128)[0]
        kb = ni.kv_bits(SEED, layer, ni.KIND_K, 1, 0, int(ctx[1]), hkv, 128)
        vb = ni.kv_bits(SEED, layer, ni.KIND_V, 1, 0, int(ctx[1]), hkv, 128)
        ref = orc.decode_attention(qb, kb, vb, np.float32(1 / np.sqrt(128)))
        got = ni.bf16_bits_to_f64(outs2[layer][1].view(torch.int16).cpu().numpy().view(np.uint16))
        assert within_tol(got, ref)[0]


# ---- NEXT-1: layer-wise swap pipeline --------------------


@pytest.mark.parametrize("staging_pages", [2, 5, 64])
def test_layerwise_pipelined_swap_out_with_deferred_join(staging_pages):
    """NEO's layer-wise swapping: in a layer loop, layer l's pages are written on
    the main stream, then swapped out for layer l only on a side stream ordered
    by an event (neo_kv_swap_out_ex + NEO_SWAP_DEFER_JOIN, the next layer's
    gather overlapping this layer's D2H); one neo_kv_swap_join at the end.  The
    host record is bit-exact against the oracle's gather definition of the final
    GPU-cache, and later writes to the GPU pages (after the deferred call's
    gather) never reach the host record."""
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST
    L = 4
    pool = make_pool(L=L, npages=64, nhost=64)
    gids = pool.alloc(NEO_GPU, 40)
    sel = gids[[5, 17, 2, 33, 8, 9, 10, 11, 39, 0, 1]]
    hids = pool.alloc(NEO_HOST, 11)
    staging = torch.empty(pool.staging_bytes(staging_pages, 0, 1), dtype=torch.uint8, device="cuda")
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    view = pool.gpu_view()
    sel_t = torch.from_numpy(sel.astype(np.int64)).cuda()
    expect = []
    for l in range(L):
        # "compute" layer l's KV on the main stream (a write to exactly those pages)
        view[l, :, sel_t] = view[l, :, sel_t] + 1 if l % 2 else view[l, :, sel_t].neg()
        expect.append(oracle.gather_pages(gpu_np(pool), sel, l, l + 1))   # syncs: the bits that must move
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        pool.swap_out(sel, hids, staging, l, l + 1, stream=side, defer_join=True)
        # once the side stream passed the call, the GPU pages may be overwritten
        done = torch.cuda.Event()
        done.record(side)
        main.wait_event(done)
        view[l, :, sel_t] = 0
    pool.swap_join(stream=side)
    side.synchronize()
    host = host_np(pool)
    for l in range(L):
        assert np.array_equal(oracle.host_record(host, hids, l, l + 1), expect[l]), l


@pytest.mark.parametrize("staging_pages", [1, 2, 3, 40])
def test_swap_out_in_multichunk_roundtrip(staging_pages):
    """Many chunks through both halves (and the one-buffer path at 1 page):
    out to host, back in to fresh ids, bit-exact."""
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST
    pool = make_pool(L=3, npages=96, nhost=40)
    old = pool.alloc(NEO_GPU, 37)
    hids = pool.alloc(NEO_HOST, 37)
    staging = torch.empty(pool.staging_bytes(staging_pages), dtype=torch.uint8, device="cuda")
    before = gpu_np(pool)
    side = torch.cuda.Stream()
    pool.swap_out(old, hids, staging, stream=side)
    side.synchronize()
    assert np.array_equal(oracle.host_record(host_np(pool), hids, 0, 3), oracle.gather_pages(before, old, 0, 3))
    new = pool.alloc(NEO_GPU, 37)
    pool.gpu_view()[:, :, torch.from_numpy(new.astype(np.int64)).cuda()] = 0
    torch.cuda.synchronize()
    pool.swap_in(hids, new, staging, stream=side)
    side.synchronize()
    after = gpu_np(pool)
    assert np.array_equal(oracle.gather_pages(after, new, 0, 3), oracle.gather_pages(before, old, 0, 3))


def test_swap_out_inside_cuda_graph():
    """Graph capture takes the one-buffer path (no cross-call events); replay is bit-exact."""
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST
    pool = make_pool()
    gids = pool.alloc(NEO_GPU, 20)
    hids = pool.alloc(NEO_HOST, 20)
    staging = torch.empty(pool.staging_bytes(6), dtype=torch.uint8, device="cuda")
    pool.swap_out(gids[:2], hids[:2], staging)           # the pool's pipeline exists before the capture
    torch.cuda.synchronize()
    pool.host.view(torch.int16).fill_(0x7FC0)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            pool.swap_out(gids, hids, staging, stream=s)
    torch.cuda.synchronize()
    assert (host_np(pool) == 0x7FC0).all()                # capture ran nothing
    before = gpu_np(pool)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(oracle.host_record(host_np(pool), hids, 0, 4), oracle.gather_pages(before, gids, 0, 4))


def test_swap_validation_enqueues_nothing():
    """All-or-nothing: a staging buffer in host memory, an unallocated id or a
    bad flag is rejected before anything is enqueued (the host pages keep their
    fill)."""
    import torch
    from paper_2411_01142_b200 import NEO_GPU, NEO_HOST, neo
    pool = make_pool()
    gids = pool.alloc(NEO_GPU, 8)
    hids = pool.alloc(NEO_HOST, 8)
    torch.cuda.synchronize()
    host_stg = torch.empty(pool.staging_bytes(8), dtype=torch.uint8).pin_memory()
    with pytest.raises(neo.NeoError):
        pool.swap_out(gids, hids, host_stg)
    stg = torch.empty(pool.staging_bytes(8), dtype=torch.uint8, device="cuda")
    with pytest.raises(neo.NeoError):
        pool.swap_out(np.append(gids[:7], 63), hids, stg)
    L = neo.lib()
    g, h = np.ascontiguousarray(gids), np.ascontiguousarray(hids)
    assert L.neo_kv_swap_out_ex(pool.handle, 8, g.ctypes.data, h.ctypes.data, 0, 4, stg.data_ptr(),
                                stg.numel(), 2, 0) == neo.NEO_ERR_INVALID_ARG
    torch.cuda.synchronize()
    assert (host_np(pool) == 0x7FC0).all()
