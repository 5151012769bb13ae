"""NEXT-2: CPU paged decode attention over the CPU-cache (neo_cpu_decode_attn,
NEO's PACPU) against the fp64 oracle, on CPU.  Same tolerance rule
as the GPU path; bitwise checks where the arithmetic is exact."""
import math

import numpy as np
import pytest

import neo_inputs as ni
import oracle
from harness import within_tol
from paper_2411_01142_b200 import neo

D = 128


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2411_01142_b200 import build
    build.build()


class HostCase:
    """Requests' KV scattered over a CPU-cache [NH][L][2][Hkv][P][D] (numpy)."""

    def __init__(self, ctx, hq, hkv, P=16, L=2, layer=1, seed=3, variant=0, extra=5):
        self.ctx = np.asarray(ctx, dtype=np.int32)
        self.hq, self.hkv, self.P, self.L, self.layer, self.seed = hq, hkv, P, L, layer, seed
        self.table, self.nh = ni.block_tables(seed, self.ctx, P, num_pages=int(ni.pages_needed(self.ctx, P).sum()) + extra)
        self.host = np.full((self.nh, L, 2, hkv, P, D), 0x7FC0, dtype=np.uint16)    # NaN poison everywhere
        self.q = ni.q_bits(seed, layer, np.arange(len(self.ctx)), hq, D, variant=variant)
        self.k, self.v = [], []
        for b, n in enumerate(self.ctx):
            kb = ni.kv_bits(seed, layer, ni.KIND_K, b, 0, int(n), hkv, D, variant=variant, hq_total=hq)
            vb = ni.kv_bits(seed, layer, ni.KIND_V, b, 0, int(n), hkv, D)
            self.k.append(kb)
            self.v.append(vb)
            for j in range((int(n) + P - 1) // P):
                t0, t1 = j * P, min(int(n), (j + 1) * P)
                pid = self.table[b, j]
                self.host[pid, layer, 0, :, :t1 - t0] = kb[t0:t1].transpose(1, 0, 2)
                self.host[pid, layer, 1, :, :t1 - t0] = vb[t0:t1].transpose(1, 0, 2)
        self.pool = neo.KVPool(L, hkv, num_gpu_pages=1, num_host_pages=self.nh, page_size=P, allocate=False,
                               host_array=self.host)

    def run(self, threads=0):
        return self.pool.cpu_decode_attn(self.layer, self.q, self.table, self.ctx, num_threads=threads)

    def check(self, out):
        got = ni.bf16_bits_to_f64(out)
        worst = 0.0
        for b in range(len(self.ctx)):
            if self.ctx[b] == 0:
                assert (got[b] == 0).all()
                continue
            ref = oracle.decode_attention(self.q[b], self.k[b], self.v[b], np.float32(1 / math.sqrt(D)))
            ok, r = within_tol(got[b], ref)
            worst = max(worst, r)
            assert ok, f"b={b} ctx={self.ctx[b]} err/tol={r:.3f}"
        return worst


@pytest.mark.parametrize("hq,hkv", [(32, 8), (64, 8), (32, 32), (8, 1), (16, 8), (28, 4), (24, 8)])
@pytest.mark.parametrize("threads", [1, 3, 8])
@pytest.mark.parametrize("path", ["2", "1", "0"])      # AVX-512 BF16 / AVX-512F / portable
def test_cpu_attn_parity(hq, hkv, threads, path, monkeypatch):
    monkeypatch.setenv("NEO_CPU_PATH", path)
    c = HostCase([1, 15, 16, 17, 33, 300, 0, 601], hq, hkv, seed=hq + threads)
    c.check(c.run(threads))


@pytest.mark.parametrize("P", [32, 64])
@pytest.mark.parametrize("path", ["2", "0"])
def test_cpu_attn_page_sizes(P, path, monkeypatch):
    monkeypatch.setenv("NEO_CPU_PATH", path)
    c = HostCase([1, 31, 32, 33, 200], 32, 8, P=P, seed=P)
    c.check(c.run(4))


@pytest.mark.parametrize("variant", [ni.VARIANT_PEAKED, ni.VARIANT_SINK])
def test_cpu_attn_variants(variant):
    c = HostCase([5, 700, 1500], 32, 8, variant=variant, seed=9)
    c.check(c.run(5))


@pytest.mark.parametrize("path", ["2", "1", "0"])
def test_cpu_attn_single_token_bitwise_and_determinism(path, monkeypatch):
    monkeypatch.setenv("NEO_CPU_PATH", path)
    c = HostCase([1, 1], 32, 8, seed=4)
    out = c.run(2)
    for b in range(2):
        for h in range(32):
            assert np.array_equal(out[b, h], c.v[b][0, h // 4])
    c2 = HostCase([100, 1234, 57], 64, 8, seed=5)
    a, b = c2.run(3), c2.run(3)
    assert np.array_equal(a, b)


def test_cpu_attn_bad_host_ids():
    c = HostCase([40], 32, 8, seed=6)
    bad = c.table.copy()
    bad[0, 1] = c.nh + 3
    with pytest.raises(neo.NeoError) as e:
        c.pool.cpu_decode_attn(c.layer, c.q, bad, c.ctx)
    assert e.value.status == neo.NEO_ERR_INVALID_ARG


def test_cpu_attn_random_configs():
    rng = np.random.default_rng(7)
    for trial in range(40):
        G = int(rng.choice([1, 2, 4, 8]))
        hkv = int(rng.choice([1, 2, 8]))
        ctx = rng.integers(0, 400, size=int(rng.integers(1, 5)))
        c = HostCase(ctx, hkv * G, hkv, P=int(rng.choice([16, 32])), seed=100 + trial)
        c.check(c.run(int(rng.integers(1, 9))))
