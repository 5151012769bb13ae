"""The device generator writes the same bits as the host generator (so the
oracle and the GPU see identical inputs at any size)."""
import numpy as np
import pytest

import neo_inputs as ni

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_01142_b200 import build
    build.build()


def test_counter_bits_host_equals_device():
    from neo_inputs import device as gen
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 1 << 40, size=200000, dtype=np.uint64)
    for tid in (1, 2, 3, 2 + 8 * 31):
        assert np.array_equal(gen.values(ni.DEFAULT_SEED, tid, idx), ni.counter_bits(ni.DEFAULT_SEED, tid, idx))


@pytest.mark.parametrize("variant", [0, ni.VARIANT_PEAKED | ni.VARIANT_SINK])
def test_fill_kv_and_q_match_host(variant):
    import torch
    from neo_inputs import device as gen
    hq, hkv, P = 32, 8, 16
    ctx = np.array([1, 16, 17, 300], dtype=np.int32)
    table, npages = ni.block_tables(3, ctx, P, num_pages=40)
    k = torch.zeros(npages, hkv, P, 128, dtype=torch.bfloat16, device="cuda")
    v = torch.zeros_like(k)
    bt, sl = torch.from_numpy(table).cuda(), torch.from_numpy(ctx).cuda()
    gen.fill_kv(k, v, bt, sl, seed=9, layer=5, hq_total=hq, b_offset=7, variant=variant, tail=gen.TAIL_NAN)
    q = torch.empty(4, hq, 128, dtype=torch.bfloat16, device="cuda")
    gen.fill_q(q, seed=9, layer=5, b_offset=7, variant=variant)
    torch.cuda.synchronize()
    assert np.array_equal(q.view(torch.int16).cpu().numpy().view(np.uint16),
                          ni.q_bits(9, 5, np.arange(4) + 7, hq, 128, variant=variant))
    kn = k.view(torch.int16).cpu().numpy().view(np.uint16)
    vn = v.view(torch.int16).cpu().numpy().view(np.uint16)
    for b in range(4):
        n = int(ctx[b])
        kb = ni.kv_bits(9, 5, ni.KIND_K, b + 7, 0, n, hkv, 128, variant=variant, hq_total=hq)
        vb = ni.kv_bits(9, 5, ni.KIND_V, b + 7, 0, n, hkv, 128)
        for t in range(n):
            pid, s = table[b, t // P], t % P
            assert np.array_equal(kn[pid, :, s], kb[t]) and np.array_equal(vn[pid, :, s], vb[t])
        if n % P:
            pid = table[b, n // P]
            assert (kn[pid, :, n % P:] == 0x7FC0).all()
