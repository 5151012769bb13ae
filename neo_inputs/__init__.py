"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO attention arithmetic (no dot products, softmax, merge or
page gather): it only produces bit patterns and integer metadata, so both sides
of every parity check can draw identical inputs from it (DESIGN.md "Input
recipe"; SURVEY.md §8(d) "Synthetic inputs").

Counter-based values (host side here, device side in ``csrc/neo_gen.cu``; a
GPU test asserts the two agree bit for bit):

    x    = splitmix64(seed ^ (tensor_id << 40) ^ index)
    s    = sum_{i=0..3} ((x >> 16 i) & 0xFFFF) - 131070      (exact int, |s| < 2^18)
    f    = s * 2^-15                                           (exact fp32)
    bf16 = round-to-nearest-even(f)                            (integer ops)

``tensor_id = kind + 8 * layer`` with kind Q=1, K=2, V=3.  Element indices:

    Q[b][h][d]        -> (b * Hq_total + h) * D + d
    K/V[b][t][g][d]   -> ((b * 2^17 + t) * Hkv_total + g) * D + d

so a request's values do not depend on the batch it is placed in, on the page
it lands in, or on how heads are sharded across ranks (b, h, g are GLOBAL ids).

Variants:
  * ``peaked``: q multiplied by 8 (exact in bf16), logit std ~10.
  * ``sink``  : K[b][t=0][g][:] = 4 * sign(sum_r q[b][g*G + r][:]) computed on
    exact integers (bf16 * 2^22), sign(0) = +1.  Gives every head of the group a
    large positive logit on token 0 (StreamingLLM-style sink).

Context lengths use numpy's PCG64 with the given seed:
  * ``uniform``  : U_int[ceil(0.9 l), floor(1.1 l)]  (§5.1 synthetic
    workloads; integer rounding per S:120).
  * ``lognormal``: median m, sigma, clipped (skewed variant).
  * ``loguniform``: floor(exp(U[ln lo, ln hi])) (config 5).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
KIND_Q, KIND_K, KIND_V = 1, 2, 3
T_STRIDE = 1 << 17          # max tokens per request in the index formula
INDEX_LIMIT = 1 << 40
VARIANT_PEAKED = 1
VARIANT_SINK = 2
DEFAULT_SEED = 0x4E454F     # bytes of "NEO"


def tensor_id(kind: int, layer: int) -> int:
    return int(kind) + 8 * int(layer)


def splitmix64(z):
    """splitmix64 output function applied to state ``z`` (Steele, Lea, Flood 2014;
    the reference generator returns splitmix64(s0 + k*gamma) for k = 1, 2, ...)."""
    z = (np.asarray(z, dtype=np.uint64) + GOLDEN_GAMMA)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 to nearest even with integer ops (finite inputs)."""
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    return ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(bits).astype(np.float64)


def counter_bits(seed: int, tid: int, index) -> np.ndarray:
    """bf16 bit patterns for element ``index`` of tensor ``tid``."""
    index = np.asarray(index, dtype=np.uint64)
    if index.size and int(index.max()) >= INDEX_LIMIT:
        raise ValueError("element index exceeds 2^40")
    x = splitmix64(np.uint64(seed) ^ (np.uint64(tid) << np.uint64(40)) ^ index)
    s = np.zeros(x.shape, dtype=np.int64)
    for i in range(4):
        s += ((x >> np.uint64(16 * i)) & np.uint64(0xFFFF)).astype(np.int64)
    s -= 131070
    f = s.astype(np.float32) * np.float32(2.0 ** -15)
    return f32_to_bf16_bits(f)


def _times8(bits: np.ndarray) -> np.ndarray:
    return f32_to_bf16_bits(bf16_bits_to_f32(bits) * np.float32(8.0))


_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "csrc", "neo_gen_host.c")
_CLIB = os.path.join(_HERE, "libneo_gen_host.so")
_clib = None
_clock = threading.Lock()


def _host_lib():
    """C version of the generator (same bits, ~100x faster than numpy)."""
    global _clib
    with _clock:
        if _clib is None:
            if not os.path.exists(_CLIB) or os.path.getmtime(_CLIB) < os.path.getmtime(_CSRC):
                tmp = _CLIB + f".tmp{os.getpid()}"
                subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _CSRC, "-lm"])
                os.replace(tmp, _CLIB)
            L = ctypes.CDLL(_CLIB)
            P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
            L.gen_q_bits.argtypes = [u64, i32, P, i32, i32, i32, i32, i32, i32, P]
            L.gen_kv_bits.argtypes = [u64, i32, i32, i64, i64, i64, i32, i32, i32, i32, i32, i32, P]
            L.gen_q_bits.restype = None
            L.gen_kv_bits.restype = None
            _clib = L
    return _clib


def _contiguous_range(heads):
    h = np.asarray(heads)
    return h.ndim == 1 and len(h) > 0 and np.array_equal(h, np.arange(h[0], h[0] + len(h)))


def q_bits(seed: int, layer: int, b_ids, hq_total: int, d: int, heads=None,
           variant: int = 0, use_c: bool = True) -> np.ndarray:
    """Q[b][h][d] bits for global requests ``b_ids`` and global heads ``heads``."""
    if use_c and (heads is None or _contiguous_range(heads)):
        b = np.ascontiguousarray(np.asarray(b_ids, dtype=np.int64).reshape(-1))
        h0, nh = (0, hq_total) if heads is None else (int(heads[0]), len(heads))
        out = np.empty((len(b), nh, d), dtype=np.uint16)
        _host_lib().gen_q_bits(seed, layer, b.ctypes.data, len(b), hq_total, h0, nh, d, variant, out.ctypes.data)
        return out
    b_ids = np.asarray(b_ids, dtype=np.uint64).reshape(-1)
    heads = np.arange(hq_total) if heads is None else np.asarray(heads)
    heads = heads.astype(np.uint64)
    dd = np.arange(d, dtype=np.uint64)
    idx = (b_ids[:, None, None] * np.uint64(hq_total) + heads[None, :, None]) * np.uint64(d) + dd
    bits = counter_bits(seed, tensor_id(KIND_Q, layer), idx)
    if variant & VARIANT_PEAKED:
        bits = _times8(bits)
    return bits


def _sink_row_bits(seed, layer, b, g, group, hq_total, d) -> np.ndarray:
    """4*sign(sum of the group's q rows) per dim, on exact integers."""
    heads = np.arange(g * group, (g + 1) * group)
    qb = q_bits(seed, layer, [b], hq_total, d, heads=heads, use_c=False)[0]   # [G][D]
    qi = np.rint(bf16_bits_to_f64(qb) * 2.0 ** 22).astype(np.int64)   # exact
    tot = qi.sum(axis=0)
    four, mfour = 0x4080, 0xC080                                       # bf16 +4, -4
    return np.where(tot >= 0, four, mfour).astype(np.uint16)


def kv_bits(seed: int, layer: int, kind: int, b: int, t_begin: int, t_end: int,
            hkv_total: int, d: int, heads=None, variant: int = 0,
            hq_total: int | None = None, use_c: bool = True) -> np.ndarray:
    """Unpaged K or V bits ``[t_end - t_begin][len(heads)][d]`` for request ``b``."""
    if t_end > T_STRIDE:
        raise ValueError("context longer than 2^17 tokens")
    if use_c and (heads is None or _contiguous_range(heads)):
        g0, ng = (0, hkv_total) if heads is None else (int(heads[0]), len(heads))
        if kind == KIND_K and (variant & VARIANT_SINK):
            assert hq_total is not None and hq_total % hkv_total == 0
        out = np.empty((max(t_end - t_begin, 0), ng, d), dtype=np.uint16)
        _host_lib().gen_kv_bits(seed, layer, kind, b, t_begin, t_end, hkv_total, g0, ng, d,
                                variant if kind == KIND_K else 0, hq_total or hkv_total, out.ctypes.data)
        return out
    heads = np.arange(hkv_total) if heads is None else np.asarray(heads)
    t = np.arange(t_begin, t_end, dtype=np.uint64)
    if t_end > T_STRIDE:
        raise ValueError("context longer than 2^17 tokens")
    hh = heads.astype(np.uint64)
    dd = np.arange(d, dtype=np.uint64)
    idx = ((np.uint64(b) * np.uint64(T_STRIDE) + t[:, None, None]) * np.uint64(hkv_total)
           + hh[None, :, None]) * np.uint64(d) + dd
    bits = counter_bits(seed, tensor_id(kind, layer), idx)
    if kind == KIND_K and (variant & VARIANT_SINK) and t_begin == 0 and t_end > 0:
        assert hq_total is not None and hq_total % hkv_total == 0
        group = hq_total // hkv_total
        for j, g in enumerate(heads):
            bits[0, j, :] = _sink_row_bits(seed, layer, b, int(g), group, hq_total, d)
    return bits


# ---------------------------------------------------------------- metadata


def ctx_uniform(seed: int, n: int, l: int) -> np.ndarray:
    """U_int[ceil(0.9 l), floor(1.1 l)]."""
    lo, hi = (9 * l + 9) // 10, (11 * l) // 10
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi + 1, size=n, dtype=np.int64).astype(np.int32)


def ctx_range(seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi + 1, size=n, dtype=np.int64).astype(np.int32)


def ctx_lognormal(seed: int, n: int, median: float, sigma: float, lo: int, hi: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.floor(median * np.exp(sigma * rng.standard_normal(n)))
    return np.clip(x, lo, hi).astype(np.int32)


def ctx_loguniform(seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.floor(np.exp(rng.uniform(math.log(lo), math.log(hi), size=n)))
    return np.clip(x, lo, hi).astype(np.int32)


def pages_needed(ctx: np.ndarray, page_size: int) -> np.ndarray:
    return (np.asarray(ctx, dtype=np.int64) + page_size - 1) // page_size


def block_tables(seed: int, ctx: np.ndarray, page_size: int, num_pages: int | None = None,
                 pad: int = 0, fill: int = -1):
    """Scatter each request's logical pages over a seeded random permutation of
    the pool (no locality, like a long-running server).  Returns
    ``(table[B][max_blocks] int32, num_pages)``; unused entries hold ``fill``."""
    need = pages_needed(ctx, page_size)
    total = int(need.sum())
    num_pages = max(total, 1) if num_pages is None else num_pages
    if num_pages < total:
        raise ValueError("pool too small")
    rng = np.random.Generator(np.random.PCG64(seed ^ 0xB10C))
    perm = rng.permutation(num_pages).astype(np.int32)
    max_blocks = int(need.max()) + pad if len(need) else pad
    max_blocks = max(max_blocks, 1)
    table = np.full((len(ctx), max_blocks), fill, dtype=np.int32)
    off = 0
    for i, n in enumerate(need):
        table[i, :n] = perm[off:off + n]
        off += n
    return table, num_pages
