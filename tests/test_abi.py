"""C-ABI checks that need no GPU: every symbol include/neo.h declares is
exported by libneo.so, argument validation returns the documented status
without touching CUDA, and the two-pool page allocator keeps S:290-293's
properties (conservation, atomicity, residency) under 10^5 random ops."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2411_01142_b200 import neo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2411_01142_b200 import build
    build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "neo.h")).read()
    return sorted(set(re.findall(r"NEO_API\s+[\w\s\*]+?\b(neo_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 16
    L = neo.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(neo.EXPORTED) == names


def test_version_and_error_text():
    assert b"sm_100a" in neo.lib().neo_version()
    with pytest.raises(neo.NeoError) as e:
        neo.workspace_bytes(4, 30, 8, 100)                 # 30 % 8 != 0
    assert e.value.status == neo.NEO_ERR_INVALID_ARG
    assert "multiple" in str(e.value)


def _attn(**kw):
    args = dict(q=16, k=16, v=16, stride=2048 * 8, npages=10, bt=16, maxb=4, sl=16, out=16, B=2, hq=32, hkv=8,
                d=128, P=16, msl=64, scale=0.088, C=0, ws=16, wsb=1 << 20, stream=0)
    args.update(kw)
    a = args
    return neo.lib().neo_decode_attn(a["q"], a["k"], a["v"], a["stride"], a["npages"], a["bt"], a["maxb"], a["sl"],
                                     a["out"], a["B"], a["hq"], a["hkv"], a["d"], a["P"], a["msl"],
                                     ctypes.c_float(a["scale"]), a["C"], a["ws"], a["wsb"], a["stream"])


@pytest.mark.parametrize("kw,status", [
    (dict(d=64), neo.NEO_ERR_UNSUPPORTED),
    (dict(P=8), neo.NEO_ERR_UNSUPPORTED),
    (dict(hq=30), neo.NEO_ERR_INVALID_ARG),
    (dict(hq=128, hkv=8), neo.NEO_ERR_UNSUPPORTED),            # G = 16
    (dict(q=0), neo.NEO_ERR_INVALID_ARG),
    (dict(q=24), neo.NEO_ERR_INVALID_ARG),                     # misaligned
    (dict(stride=2048 * 8 - 8), neo.NEO_ERR_INVALID_ARG),      # page stride < Hkv*P*D
    (dict(msl=65), neo.NEO_ERR_INVALID_ARG),                   # > max_blocks * P
    (dict(wsb=16), neo.NEO_ERR_INVALID_ARG),                   # workspace too small
    (dict(C=24), neo.NEO_ERR_UNSUPPORTED),
    (dict(C=1040), neo.NEO_ERR_UNSUPPORTED),                   # > 1024
    (dict(scale=0.0), neo.NEO_ERR_INVALID_ARG),
    (dict(npages=0), neo.NEO_ERR_INVALID_ARG),
])
def test_decode_attn_validation(kw, status):
    assert _attn(**kw) == status


def test_decode_attn_batch_zero_is_noop():
    assert _attn(B=0, q=0, out=0) == neo.NEO_OK


def _prefill(**kw):
    a = dict(q=16, k=16, v=16, stride=2048 * 8, npages=10, bt=16, maxb=4, sl=16, qo=16, out=16, B=2, T=100, hq=32,
             hkv=8, d=128, P=16, mql=64, scale=0.088, stream=0)
    a.update(kw)
    return neo.lib().neo_prefill_attn(a["q"], a["k"], a["v"], a["stride"], a["npages"], a["bt"], a["maxb"], a["sl"],
                                      a["qo"], a["out"], a["B"], a["T"], a["hq"], a["hkv"], a["d"], a["P"], a["mql"],
                                      ctypes.c_float(a["scale"]), a["stream"])


@pytest.mark.parametrize("kw,status", [
    (dict(d=64), neo.NEO_ERR_UNSUPPORTED),
    (dict(P=24), neo.NEO_ERR_UNSUPPORTED),
    (dict(hq=30), neo.NEO_ERR_INVALID_ARG),
    (dict(hq=24, hkv=8), neo.NEO_ERR_UNSUPPORTED),             # G = 3
    (dict(hq=256, hkv=8), neo.NEO_ERR_UNSUPPORTED),            # G = 32
    (dict(B=513), neo.NEO_ERR_UNSUPPORTED),                    # schedule table limit
    (dict(mql=65537), neo.NEO_ERR_UNSUPPORTED),                # max_q_len * G > 262144
    (dict(q=0), neo.NEO_ERR_INVALID_ARG),
    (dict(qo=0), neo.NEO_ERR_INVALID_ARG),
    (dict(out=24), neo.NEO_ERR_INVALID_ARG),                   # misaligned
    (dict(stride=2048 * 8 - 8), neo.NEO_ERR_INVALID_ARG),
    (dict(mql=0), neo.NEO_ERR_INVALID_ARG),
    (dict(scale=float("nan")), neo.NEO_ERR_INVALID_ARG),
])
def test_prefill_attn_validation(kw, status):
    assert _prefill(**kw) == status


def test_prefill_attn_empty_is_noop():
    assert _prefill(B=0, q=0, out=0) == neo.NEO_OK
    assert _prefill(T=0, q=0, out=0) == neo.NEO_OK


def test_workspace_bytes_and_default_chunk():
    assert neo.default_chunk(256, 8, 1126) == 512
    assert neo.default_chunk(512, 1, 2252) == 256
    assert neo.default_chunk(128, 8, 8192) == 512
    assert neo.default_chunk(4, 32, 128) == 64
    # single chunk: counters only; split: counters + (m, l) + fp32 partials.  The
    # counter region is size/64 (fixed by the workspace size) and must hold B*Hkv ints.
    small = neo.workspace_bytes(4, 32, 32, 64, chunk_tokens=64)
    assert small // 64 >= 4 * 32 * 4
    big = neo.workspace_bytes(256, 32, 8, 1126, chunk_tokens=256)
    units = 256 * 8 * 5
    data = units * 4 * 8 + units * 4 * 128 * 4
    assert big >= data + 256 * 8 * 4 and (big // 64) & ~255 >= 256 * 8 * 4
    assert big <= 1.05 * data + 65536


def _plan_replay(ctx, hkv, P, sms=148, o=6.0, og=2.0, om=2.0):
    """Independent replay of the planner's model (include/neo.h
    neo_decode_attn_plan_chunk): split-K units in chunk-major order, W = 4 per CTA,
    CTAs taken in order by the earliest-free slot (SMs x CTAs/SM of the default
    shape); the grouped kernel's CTAs likewise at 3 per SM.  None = latency-bound
    (library default)."""
    import heapq
    nt = [(c + 15) // 16 for c in ctx]
    cands = [C for C in (1024, 640, 512, 448, 384, 320, 256) if C % P == 0] or [P]

    def shape(mc):
        return (4, 2) if mc <= 3 else (4, 3)          # (warps, CTAs/SM)

    def split_score(C):
        ct = C // 16
        mc = max([-(-t // ct) for t in nt] + [1])
        w, k = shape(mc)
        units = [min(max(t - c * ct, 0), ct) for c in range(mc) for t in nt for _ in range(hkv)]
        units += [0] * (-len(units) % w)
        heap = [0.0] * (sms * k)
        for i in range(0, len(units), w):
            m = max(units[i:i + w])
            if m:
                heapq.heapreplace(heap, heap[0] + o + m)
        return sum(nt) * hkv / max(heap)

    def grouped_score(gt):
        heap = [0.0] * (sms * 3)
        mg = max([-(-t // gt) for t in nt] + [1])
        order = [(q, t) for t in nt for q in range(mg)] if mg >= 3 else [(q, t) for q in range(mg) for t in nt]
        for q, t in order:
            ng = -(-t // gt)
            if q >= ng:
                continue
            tg = -(-t // ng)
            g0, g1 = q * tg, min(q * tg + tg, t)
            for _ in range(hkv):
                heapq.heapreplace(heap, heap[0] + og + -(-(g1 - g0) // 4) + (om if ng > 1 else 0.0))
        return sum(nt) * hkv / max(heap)

    ctn = cands[-1] // 16
    if sum(hkv * -(-t // ctn) for t in nt) < sms * 8:
        return -1 if 0 < max(ctx) <= 4096 else None   # latency-bound: grouped, else library default
    ct0 = cands[0] // 16
    units = sum(hkv * -(-t // ct0) for t in nt)
    w, k = shape(max([-(-t // ct0) for t in nt] + [1]))
    if units >= 16 * sms * k * w:
        best, best_sc = cands[0], split_score(cands[0])
    else:
        best, best_sc = cands[0], -1.0
        for C in cands:
            sc = split_score(C)
            if sc > best_sc * 1.01:
                best, best_sc = C, sc
    best_g, best_t = -1.0, 0
    for T in (4096, 3072, 2048, 1536, 1024):
        sc = grouped_score(T // 16)
        if sc > best_g * 1.01:
            best_g, best_t = sc, T
    code = {4096: -1, 2048: -2, 1024: -4}.get(best_t, -best_t)
    return code if best_g > best_sc * 1.01 else best


def test_plan_chunk():
    """a0 planner: valid chunks, >= 4 waves -> 512, measured c4-shard picks, and
    agreement with an independent replay of its dispatch model."""
    from neo_inputs.workloads import WORKLOADS
    rng = np.random.default_rng(307)
    for _ in range(40):
        B, hkv, P = int(rng.integers(1, 700)), int(rng.choice([1, 2, 4, 8])), int(rng.choice([16, 32, 64]))
        ctx = rng.integers(0, int(rng.choice([300, 3000, 20000])), size=B).astype(np.int32)
        C = neo.plan_chunk(ctx, hkv, P)
        assert C in (-1, -2, -4, -3072, -1536) or (C % 16 == 0 and C % P == 0 and 16 <= C <= 1024)
        ref = _plan_replay(ctx.tolist(), hkv, P)
        if ref is not None:
            assert C == ref, (B, hkv, P, C, ref)
    c5 = WORKLOADS["c5"].contexts()
    assert neo.plan_chunk(c5, 8, 16) == neo.NEO_CHUNK_GROUPED    # profiles/r01_grouped_sweep.txt: +3.3 %
    c4 = WORKLOADS["c4"].contexts()
    # the c4 shards: uniform ~2K contexts -> grouped kernel, with smaller groups as
    # the per-rank (request, head) count falls (profiles/r01_grouped_sweep.txt)
    assert [neo.plan_chunk(c4, 8 // n, 16) for n in (8, 4, 2, 1)] == [-2, -2, -1, -1]
    # uniform ~1K batches of 2048 (request, kv-head) pairs take the grouped kernel (c2)
    assert neo.plan_chunk(WORKLOADS["c2"].contexts(), 8, 16) == neo.NEO_CHUNK_GROUPED
    # c3 (4K-8K): 3072-token groups (profiles/r02_group_sweep.md: 6931-6963 GB/s vs 6719-6960 for split 640)
    assert neo.plan_chunk(WORKLOADS["c3"].contexts(), 8, 16) == -3072
    assert neo.plan_chunk([], 8, 16) == neo.default_chunk(0, 8, 0)
    assert neo.plan_chunk(WORKLOADS["c1"].contexts(), 32, 16) == neo.NEO_CHUNK_GROUPED   # latency-bound c1
    with pytest.raises(neo.NeoError) as e:
        neo.plan_chunk([5, -1], 8, 16)
    assert e.value.status == neo.NEO_ERR_INVALID_ARG
    with pytest.raises(neo.NeoError) as e:
        neo.plan_chunk([5], 8, 24)
    assert e.value.status == neo.NEO_ERR_UNSUPPORTED
    with pytest.raises(neo.NeoError) as e:
        neo.plan_chunk([5], 0, 16)
    assert e.value.status == neo.NEO_ERR_INVALID_ARG


def test_grouped_workspace_and_chunk_validation():
    """NEO_CHUNK_GROUPED: requests <= 4096 tokens need no partials (counters only);
    longer ones one partial row set per 4096-token group.  Other negatives are invalid."""
    one = neo.workspace_bytes(256, 32, 8, 1126, chunk_tokens=neo.NEO_CHUNK_GROUPED)
    three = neo.workspace_bytes(256, 32, 8, 9000, chunk_tokens=neo.NEO_CHUNK_GROUPED)
    assert one < 256 * 8 * 4 * 64 * 2                      # counter region only
    units = 256 * 8 * 3
    assert three >= units * 4 * 8 + units * 4 * 128 * 4
    four = neo.workspace_bytes(256, 32, 8, 4096, chunk_tokens=-4)   # 1024-token groups: 4 per request
    assert four >= 256 * 8 * 4 * (4 * 8 + 4 * 128 * 4)
    # any group of T tokens, T a multiple of 16 in [64, 4096]: -1536 -> 3 groups of a 4096-token request
    t1536 = neo.workspace_bytes(256, 32, 8, 4096, chunk_tokens=-1536)
    assert t1536 >= 256 * 8 * 3 * (4 * 8 + 4 * 128 * 4)
    assert neo.workspace_bytes(256, 32, 8, 4096, chunk_tokens=-4096) == neo.workspace_bytes(
        256, 32, 8, 4096, chunk_tokens=-1)
    for bad in (-3, -5, -48, -1000, -4112, -8192):
        with pytest.raises(neo.NeoError) as e:
            neo.workspace_bytes(256, 32, 8, 1126, chunk_tokens=bad)
        assert e.value.status == neo.NEO_ERR_UNSUPPORTED, bad
    assert _attn(C=-1) != neo.NEO_ERR_UNSUPPORTED           # accepted (fails later only on fake pointers)
    assert _attn(C=-768) != neo.NEO_ERR_UNSUPPORTED


def test_pool_bytes_and_layer_view():
    pool = neo.KVPool(num_layers=3, num_kv_heads=8, num_gpu_pages=10, num_host_pages=4, allocate=False)
    page = 8 * 16 * 128 * 2
    assert pool.gpu_bytes == 3 * 2 * 10 * page
    assert pool.host_bytes == 3 * 2 * 4 * page
    pool.close()
    # layer view pointer arithmetic on a fake (never dereferenced) base
    geo = neo.Geometry(3, 8, 128, 16, 10, 0)
    h = ctypes.c_void_p()
    base = 1 << 32
    neo.check(neo.lib().neo_kv_pool_create(ctypes.byref(geo), base, 3 * 2 * 10 * page, None, 0, ctypes.byref(h)))
    k, v, s = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    neo.check(neo.lib().neo_kv_layer_view(h, 2, ctypes.byref(k), ctypes.byref(v), ctypes.byref(s)))
    assert k.value == base + 4 * 10 * page and v.value == base + 5 * 10 * page and s.value == 8 * 16 * 128
    assert neo.lib().neo_kv_layer_view(h, 3, ctypes.byref(k), ctypes.byref(v), ctypes.byref(s)) == 1
    neo.lib().neo_kv_pool_destroy(h)


def test_pool_create_validation():
    geo = neo.Geometry(1, 8, 128, 16, 10, 2)
    h = ctypes.c_void_p()
    L = neo.lib()
    assert L.neo_kv_pool_create(ctypes.byref(geo), 1 << 32, 1, 1 << 33, 1 << 30, ctypes.byref(h)) == 1  # small
    assert L.neo_kv_pool_create(ctypes.byref(geo), (1 << 32) + 8, 1 << 30, 1 << 33, 1 << 30,
                                ctypes.byref(h)) == 1                                                   # misaligned
    assert L.neo_kv_pool_create(ctypes.byref(geo), 1 << 32, 1 << 30, None, 1 << 30, ctypes.byref(h)) == 1
    bad = neo.Geometry(1, 8, 96, 16, 10, 2)
    assert L.neo_kv_pool_create(ctypes.byref(bad), 1 << 32, 1 << 30, 1 << 33, 1 << 30, ctypes.byref(h)) == 3


def test_allocator_examples():
    pool = neo.KVPool(1, 8, num_gpu_pages=10, num_host_pages=8, allocate=False)
    a = pool.alloc(neo.NEO_GPU, 3)
    assert pool.free_count(neo.NEO_GPU) == 7 and len(set(a)) == 3
    with pytest.raises(neo.NeoError) as e:
        pool.alloc(neo.NEO_GPU, 8)                         # free=7, need 8: state unchanged
    assert e.value.status == neo.NEO_ERR_OUT_OF_PAGES and pool.free_count(neo.NEO_GPU) == 7
    assert len(pool.alloc(neo.NEO_GPU, 0)) == 0
    h = pool.alloc(neo.NEO_HOST, 5)
    assert list(h) == [0, 1, 2, 3, 4]                      # one contiguous run
    pool.free(neo.NEO_HOST, [1, 3])
    h2 = pool.alloc(neo.NEO_HOST, 3)
    assert list(h2) == [5, 6, 7]                           # first contiguous run of 3
    h3 = pool.alloc(neo.NEO_HOST, 2)
    assert sorted(h3) == [1, 3]                            # no run: lowest free ids
    with pytest.raises(neo.NeoError):
        pool.free(neo.NEO_GPU, [a[0], a[0]])               # duplicate: nothing freed
    assert pool.free_count(neo.NEO_GPU) == 7
    with pytest.raises(neo.NeoError):
        pool.free(neo.NEO_GPU, [a[0], 9 if 9 not in a else 8])   # not allocated
    assert pool.free_count(neo.NEO_GPU) == 7
    pool.free(neo.NEO_GPU, a)
    assert pool.free_count(neo.NEO_GPU) == 10


def test_allocator_random_ops_conservation():
    """10^5 random alloc/extend/migrate/release ops over two pools."""
    rng = np.random.default_rng(0)
    G, H = 300, 500
    pool = neo.KVPool(1, 1, num_gpu_pages=G, num_host_pages=H, allocate=False)
    reqs = {}                                   # id -> (where, list of pages)
    owner = {neo.NEO_GPU: {}, neo.NEO_HOST: {}}  # page -> req
    next_id = 0
    for step in range(100000):
        op = rng.integers(0, 4)
        if op == 0 or not reqs:                 # allocate
            where = int(rng.integers(0, 2))
            n = int(rng.integers(0, 12))
            before = pool.free_count(where)
            try:
                ids = pool.alloc(where, n)
            except neo.NeoError as e:
                assert e.status == neo.NEO_ERR_OUT_OF_PAGES and before < n
                assert pool.free_count(where) == before
                continue
            for p in ids:
                assert p not in owner[where]
                owner[where][int(p)] = next_id
            reqs[next_id] = (where, [int(p) for p in ids])
            next_id += 1
        else:
            rid = list(reqs)[int(rng.integers(0, len(reqs)))]
            where, pages = reqs[rid]
            if op == 1:                         # extend by one page
                try:
                    p = int(pool.alloc(where, 1)[0])
                except neo.NeoError:
                    continue
                owner[where][p] = rid
                pages.append(p)
            elif op == 2:                       # migrate to the other pool (all-or-nothing)
                other = 1 - where
                try:
                    new = pool.alloc(other, len(pages))
                except neo.NeoError:
                    continue
                pool.free(where, pages)
                for p in pages:
                    del owner[where][p]
                for p in new:
                    owner[other][int(p)] = rid
                reqs[rid] = (other, [int(p) for p in new])
            else:                               # release
                pool.free(where, pages)
                for p in pages:
                    del owner[where][p]
                del reqs[rid]
        if step % 997 == 0:
            assert pool.free_count(neo.NEO_GPU) + len(owner[neo.NEO_GPU]) == G
            assert pool.free_count(neo.NEO_HOST) + len(owner[neo.NEO_HOST]) == H
    assert pool.free_count(neo.NEO_GPU) + len(owner[neo.NEO_GPU]) == G
    assert pool.free_count(neo.NEO_HOST) + len(owner[neo.NEO_HOST]) == H
    # residency exclusivity: each request's pages are all in one pool
    for rid, (where, pages) in reqs.items():
        assert all(owner[where][p] == rid for p in pages)


def test_swap_validation_without_gpu():
    pool = neo.KVPool(4, 8, num_gpu_pages=10, num_host_pages=10, allocate=False)
    g = pool.alloc(neo.NEO_GPU, 2)
    h = pool.alloc(neo.NEO_HOST, 2)
    L = neo.lib()
    gi, hi = np.ascontiguousarray(g), np.ascontiguousarray(h)
    per = pool.staging_bytes(1, 0, 4)
    assert per == 4 * 2 * 8 * 16 * 128 * 2
    # layer range out of bounds
    assert L.neo_kv_swap_out(pool.handle, 2, gi.ctypes.data, hi.ctypes.data, 0, 5, 16, per, 0) == 1
    # staging too small
    assert L.neo_kv_swap_out(pool.handle, 2, gi.ctypes.data, hi.ctypes.data, 0, 4, 16, per - 16, 0) == 1
    # unallocated host page
    bad = np.array([h[0], 9], dtype=np.int32)
    assert L.neo_kv_swap_out(pool.handle, 2, gi.ctypes.data, bad.ctypes.data, 0, 4, 16, per, 0) == 1
    # duplicate gpu ids
    dup = np.array([g[0], g[0]], dtype=np.int32)
    assert L.neo_kv_swap_in(pool.handle, 2, hi.ctypes.data, dup.ctypes.data, 0, 4, 16, per, 0) == 1
    assert L.neo_kv_swap_out(pool.handle, 0, None, None, 0, 4, None, 0, 0) == 0    # n = 0 no-op


def test_swap_ex_flag_validation_without_gpu():
    pool = neo.KVPool(4, 8, num_gpu_pages=10, num_host_pages=10, allocate=False)
    g = np.ascontiguousarray(pool.alloc(neo.NEO_GPU, 2))
    h = np.ascontiguousarray(pool.alloc(neo.NEO_HOST, 2))
    L = neo.lib()
    per = pool.staging_bytes(1, 0, 4)
    # unknown flag bits
    assert L.neo_kv_swap_out_ex(pool.handle, 2, g.ctypes.data, h.ctypes.data, 0, 4, 16, per, 6, 0) == 1
    # n = 0 is a no-op with the defer flag too; join without any pipelined swap is a no-op
    assert L.neo_kv_swap_out_ex(pool.handle, 0, None, None, 0, 4, None, 0, neo.NEO_SWAP_DEFER_JOIN, 0) == 0
    assert L.neo_kv_swap_join(pool.handle, 0) == 0
    assert L.neo_kv_swap_join(None, 0) == 1
