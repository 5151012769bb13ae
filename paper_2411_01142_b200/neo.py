"""Thin Python binding of libneo (include/neo.h).  Argument marshalling only:
every step of the hot path runs in the CUDA library.  torch supplies device
memory, pinned host memory and streams -- plumbing, not compute.

There is no fallback: if ``libneo.so`` is missing this module raises on first
use, and every compute entry point requires CUDA tensors.
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NEO_LIB") or os.path.join(_HERE, "libneo.so")   # NEO_LIB: A/B builds

NEO_OK, NEO_ERR_INVALID_ARG, NEO_ERR_OUT_OF_PAGES, NEO_ERR_UNSUPPORTED, NEO_ERR_CUDA, NEO_ERR_INTERNAL = range(6)
NEO_GPU, NEO_HOST = 0, 1
NEO_CHUNK_GROUPED = -1          # chunk_tokens selecting the grouped split-K kernel (include/neo.h)
NEO_SWAP_DEFER_JOIN = 1         # neo_kv_swap_out_ex flag (include/neo.h)
NEO_ATTN_KV_STABLE = 1          # neo_decode_attn_ex flag (include/neo.h)
STATUS_NAMES = {0: "NEO_OK", 1: "NEO_ERR_INVALID_ARG", 2: "NEO_ERR_OUT_OF_PAGES", 3: "NEO_ERR_UNSUPPORTED",
                4: "NEO_ERR_CUDA", 5: "NEO_ERR_INTERNAL"}

EXPORTED = ["neo_last_error", "neo_version", "neo_kv_pool_bytes", "neo_kv_pool_create", "neo_kv_pool_destroy",
            "neo_kv_alloc", "neo_kv_free", "neo_kv_free_count", "neo_kv_layer_view", "neo_decode_attn",
            "neo_decode_attn_default_chunk", "neo_decode_attn_plan_chunk", "neo_decode_attn_workspace_bytes", "neo_decode_attn_workspace_init",
            "neo_kv_swap_out", "neo_kv_swap_in", "neo_kv_swap_staging_bytes", "neo_cpu_decode_attn",
            "neo_kv_append", "neo_schedule", "neo_rope_append", "neo_prefill_append", "neo_prefill_attn",
            "neo_decode_attn_append", "neo_kv_swap_out_ex", "neo_kv_swap_join", "neo_decode_attn_ex"]


class NeoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Geometry(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("num_gpu_pages", ctypes.c_int64), ("num_host_pages", ctypes.c_int64)]


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2411_01142_b200.build` "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
            L.neo_last_error.restype = ctypes.c_char_p
            L.neo_version.restype = ctypes.c_char_p
            sig = {
                "neo_kv_pool_bytes": [P, P, P],
                "neo_kv_pool_create": [P, P, sz, P, sz, P],
                "neo_kv_alloc": [P, i32, i32, P],
                "neo_kv_free": [P, i32, i32, P],
                "neo_kv_free_count": [P, i32, P],
                "neo_kv_layer_view": [P, i32, P, P, P],
                "neo_decode_attn": [P, P, P, i64, i64, P, i32, P, P, i32, i32, i32, i32, i32, i32,
                                    ctypes.c_float, i32, P, sz, P],
                "neo_decode_attn_workspace_bytes": [i32, i32, i32, i32, i32, i32, P],
                "neo_decode_attn_workspace_init": [P, sz, P],
                "neo_kv_swap_out": [P, i32, P, P, i32, i32, P, sz, P],
                "neo_kv_swap_in": [P, i32, P, P, i32, i32, P, sz, P],
                "neo_kv_swap_out_ex": [P, i32, P, P, i32, i32, P, sz, ctypes.c_uint32, P],
                "neo_kv_swap_join": [P, P],
                "neo_decode_attn_ex": [P, P, P, i64, i64, P, i32, P, P, i32, i32, i32, i32, i32, i32,
                                       ctypes.c_float, i32, P, sz, ctypes.c_uint32, P],
                "neo_kv_swap_staging_bytes": [P, i32, i32, i32, P],
                "neo_cpu_decode_attn": [P, i32, P, P, i32, P, P, i32, i32, ctypes.c_float, i32],
                "neo_kv_append": [P, P, i64, i64, P, i32, P, P, P, i32, i32, i32, i32, P],
                "neo_schedule": [P, P, i32, i64, i64, P, P, P, P, P],
                "neo_rope_append": [P, i32, P, P, P, i64, i64, P, i32, P, P, P, i32, i32, i32, i32, P],
                "neo_decode_attn_append": [P, P, P, P, P, P, i64, i64, P, i32, P, P, i32, i32, i32, i32, i32, i32,
                                           ctypes.c_float, i32, P, sz, P],
                "neo_prefill_attn": [P, P, P, i64, i64, P, i32, P, P, P, i32, i32, i32, i32, i32, i32, i32,
                                     ctypes.c_float, P],
                "neo_prefill_append": [P, i32, P, P, P, i64, i64, P, i32, P, P, P, P, i32, i32, i32, i32, i32, P],
            }
            for name, args in sig.items():
                if os.environ.get("NEO_LIB") and not hasattr(L, name):
                    continue                      # older A/B build without this entry point
                f = getattr(L, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            L.neo_kv_pool_destroy.argtypes = [P]
            L.neo_kv_pool_destroy.restype = None
            L.neo_decode_attn_default_chunk.argtypes = [i32, i32, i32]
            L.neo_decode_attn_default_chunk.restype = i32
            L.neo_decode_attn_plan_chunk.argtypes = [ctypes.c_void_p, i32, i32, i32, ctypes.POINTER(i32)]
            L.neo_decode_attn_plan_chunk.restype = i32
            _lib = L
    return _lib


def check(status: int) -> None:
    if status != NEO_OK:
        raise NeoError(status, lib().neo_last_error().decode())


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _host_u16(t) -> np.ndarray:
    if isinstance(t, np.ndarray):
        return np.ascontiguousarray(t, dtype=np.uint16)
    import torch
    if t.is_cuda:
        raise ValueError("CPU attention takes host tensors")
    return np.ascontiguousarray(t.contiguous().view(torch.int16).numpy().view(np.uint16))


def _ids(ids) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(ids, dtype=np.int32).reshape(-1))


# ------------------------------------------------------------------ attention


def default_chunk(batch: int, num_kv_heads: int, max_seq_len: int) -> int:
    return int(lib().neo_decode_attn_default_chunk(batch, num_kv_heads, max_seq_len))


def plan_chunk(seq_lens, num_kv_heads: int, page_size: int = 16) -> int:
    """a0 plan from HOST request lengths (include/neo.h neo_decode_attn_plan_chunk)."""
    sl = _ids(seq_lens)
    out = ctypes.c_int32()
    check(lib().neo_decode_attn_plan_chunk(sl.ctypes.data if sl.size else None, int(sl.size), num_kv_heads,
                                            page_size, ctypes.byref(out)))
    return int(out.value)


def workspace_bytes(batch: int, num_q_heads: int, num_kv_heads: int, max_seq_len: int,
                    chunk_tokens: int = 0, head_dim: int = 128) -> int:
    out = ctypes.c_size_t()
    check(lib().neo_decode_attn_workspace_bytes(batch, num_q_heads, num_kv_heads, head_dim, max_seq_len,
                                                chunk_tokens, ctypes.byref(out)))
    return out.value


def make_workspace(batch: int, num_q_heads: int, num_kv_heads: int, max_seq_len: int, chunk_tokens: int = 0,
                   device=None, stream=None):
    """Allocate (torch) and initialise a decode-attention workspace."""
    import torch
    n = workspace_bytes(batch, num_q_heads, num_kv_heads, max_seq_len, chunk_tokens)
    ws = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
    check(lib().neo_decode_attn_workspace_init(ws.data_ptr(), n, _stream(stream)))
    return ws


def decode_attn(q, k_pages, v_pages, block_table, seq_lens, max_seq_len: int, *, out=None, scale=None,
                chunk_tokens: int = 0, workspace=None, stream=None, num_pages=None, kv_stable: bool = False):
    """Batched paged GQA decode attention: ``neo_decode_attn``
    (``neo_decode_attn_ex`` with NEO_ATTN_KV_STABLE when ``kv_stable``).

    q [B][Hq][D] bf16 cuda; k_pages/v_pages [num_pages][Hkv][P][D] bf16 cuda views
    (page stride taken from ``stride(0)``; inner [Hkv][P][D] must be contiguous);
    block_table [B][max_blocks] int32 cuda; seq_lens [B] int32 cuda."""
    import torch
    for name, t in (("q", q), ("k_pages", k_pages), ("v_pages", v_pages), ("block_table", block_table),
                    ("seq_lens", seq_lens)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if q.dtype != torch.bfloat16 or k_pages.dtype != torch.bfloat16 or v_pages.dtype != torch.bfloat16:
        raise ValueError("q, k_pages and v_pages must be bf16")
    if block_table.dtype != torch.int32 or seq_lens.dtype != torch.int32:
        raise ValueError("block_table and seq_lens must be int32")
    if not q.is_contiguous() or not block_table.is_contiguous() or not seq_lens.is_contiguous():
        raise ValueError("q, block_table and seq_lens must be contiguous")
    B, hq, d = q.shape
    npages, hkv, P, d2 = k_pages.shape
    if tuple(v_pages.shape) != tuple(k_pages.shape) or v_pages.stride() != k_pages.stride():
        raise ValueError("k_pages and v_pages must have the same shape and strides")
    if k_pages.stride()[1:] != (P * d2, d2, 1):
        raise ValueError("each page's [Hkv][P][D] block must be contiguous")
    if out is None:
        out = torch.empty_like(q)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if workspace is None:
        workspace = make_workspace(B, hq, hkv, max_seq_len, chunk_tokens, device=q.device, stream=stream)
    args = (q.data_ptr(), k_pages.data_ptr(), v_pages.data_ptr(), k_pages.stride(0),
            int(num_pages if num_pages is not None else npages), block_table.data_ptr(), block_table.shape[1],
            seq_lens.data_ptr(), out.data_ptr(), B, hq, hkv, d, P, int(max_seq_len), float(scale), int(chunk_tokens),
            workspace.data_ptr(), workspace.numel())
    if kv_stable:
        check(lib().neo_decode_attn_ex(*args, NEO_ATTN_KV_STABLE, _stream(stream)))
    else:
        check(lib().neo_decode_attn(*args, _stream(stream)))
    return out


def decode_attn_append(q, k_pages, v_pages, block_table, seq_lens, max_seq_len, k_new, v_new, inv_freq=None,
                       out=None, scale=None, chunk_tokens=0, workspace=None, stream=None, num_pages=None):
    """neo_decode_attn_append: one launch that RoPE-rotates q (registers only) and
    k_new at position seq_lens[b]-1 (inv_freq float32 [D/2] cuda, or None for a
    plain append), stores k/v into the page slot and attends over the grown
    context."""
    import torch
    for name, t in (("q", q), ("k_pages", k_pages), ("v_pages", v_pages), ("block_table", block_table),
                    ("seq_lens", seq_lens), ("k_new", k_new), ("v_new", v_new)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if inv_freq is not None and (not inv_freq.is_cuda or inv_freq.dtype != torch.float32):
        raise ValueError("inv_freq must be a float32 CUDA tensor")
    if not (q.is_contiguous() and k_new.is_contiguous() and v_new.is_contiguous()):
        raise ValueError("q, k_new and v_new must be contiguous")
    B, hq, d = q.shape
    npages, hkv, P, _ = k_pages.shape
    if k_pages.stride()[1:] != (P * d, d, 1) or v_pages.stride() != k_pages.stride():
        raise ValueError("each page's [Hkv][P][D] block must be contiguous, K and V alike")
    if out is None:
        out = torch.empty_like(q)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if workspace is None:
        workspace = make_workspace(B, hq, hkv, max_seq_len, chunk_tokens, device=q.device, stream=stream)
    check(lib().neo_decode_attn_append(
        q.data_ptr(), inv_freq.data_ptr() if inv_freq is not None else None, k_new.data_ptr(), v_new.data_ptr(),
        k_pages.data_ptr(), v_pages.data_ptr(), k_pages.stride(0), int(num_pages if num_pages is not None else npages),
        block_table.data_ptr(), block_table.shape[1], seq_lens.data_ptr(), out.data_ptr(), B, hq, hkv, d, P,
        int(max_seq_len), float(scale), int(chunk_tokens), workspace.data_ptr(), workspace.numel(), _stream(stream)))
    return out


def kv_append(k_pages, v_pages, block_table, seq_lens, k_new, v_new, stream=None, num_pages=None):
    """neo_kv_append: write k_new/v_new [B][Hkv][D] (bf16, cuda) at
    token seq_lens[b]-1 of each request's pages."""
    import torch
    for name, t in (("k_pages", k_pages), ("v_pages", v_pages), ("block_table", block_table), ("seq_lens", seq_lens),
                    ("k_new", k_new), ("v_new", v_new)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if k_new.dtype != torch.bfloat16 or v_new.dtype != torch.bfloat16 or not k_new.is_contiguous() \
            or not v_new.is_contiguous():
        raise ValueError("k_new / v_new must be contiguous bf16")
    npages, hkv, P, d = k_pages.shape
    check(lib().neo_kv_append(k_pages.data_ptr(), v_pages.data_ptr(), k_pages.stride(0),
                              int(num_pages if num_pages is not None else npages), block_table.data_ptr(),
                              block_table.shape[1], seq_lens.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                              k_new.shape[0], hkv, d, P, _stream(stream)))


def rope_append(q, inv_freq, k_pages, v_pages, block_table, seq_lens, k_new, v_new, stream=None, num_pages=None):
    """neo_rope_append: rotate q (in place) and k_new at position seq_lens[b]-1 with
    the frequency table inv_freq (float32 [D/2], cuda), write k/v into the pages."""
    import torch
    for name, t in (("q", q), ("inv_freq", inv_freq), ("k_pages", k_pages), ("k_new", k_new), ("v_new", v_new)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if inv_freq.dtype != torch.float32 or not q.is_contiguous():
        raise ValueError("inv_freq must be float32 and q contiguous")
    npages, hkv, P, d = k_pages.shape
    check(lib().neo_rope_append(q.data_ptr(), q.shape[1], inv_freq.data_ptr(), k_pages.data_ptr(),
                                v_pages.data_ptr(), k_pages.stride(0), int(num_pages if num_pages is not None else npages),
                                block_table.data_ptr(), block_table.shape[1], seq_lens.data_ptr(), k_new.data_ptr(),
                                v_new.data_ptr(), q.shape[0], hkv, d, P, _stream(stream)))


def prefill_attn(q, k_pages, v_pages, block_table, seq_lens, q_offsets, max_q_len, out=None, scale=None,
                 stream=None, num_pages=None):
    """neo_prefill_attn: causal attention of the packed prompt-chunk rows q
    [T][Hq][D] (bf16, cuda) over each request's paged KV; q_offsets [B+1] int32."""
    import torch
    for name, t in (("q", q), ("k_pages", k_pages), ("v_pages", v_pages), ("block_table", block_table),
                    ("seq_lens", seq_lens), ("q_offsets", q_offsets)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if q.dtype != torch.bfloat16 or not q.is_contiguous():
        raise ValueError("q must be contiguous bf16")
    if q_offsets.dtype != torch.int32 or seq_lens.dtype != torch.int32 or block_table.dtype != torch.int32:
        raise ValueError("q_offsets, seq_lens and block_table must be int32")
    T, hq, d = q.shape
    npages, hkv, P, _ = k_pages.shape
    if k_pages.stride()[1:] != (P * d, d, 1) or v_pages.stride() != k_pages.stride():
        raise ValueError("each page's [Hkv][P][D] block must be contiguous, K and V alike")
    if out is None:
        out = torch.empty_like(q)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    check(lib().neo_prefill_attn(q.data_ptr(), k_pages.data_ptr(), v_pages.data_ptr(), k_pages.stride(0),
                                 int(num_pages if num_pages is not None else npages), block_table.data_ptr(),
                                 block_table.shape[1], seq_lens.data_ptr(), q_offsets.data_ptr(), out.data_ptr(),
                                 seq_lens.shape[0], T, hq, hkv, d, P, int(max_q_len), float(scale), _stream(stream)))
    return out


def prefill_append(k_pages, v_pages, block_table, seq_lens, q_offsets, k_new, v_new, q=None, inv_freq=None,
                   stream=None, num_pages=None):
    """neo_prefill_append: store the packed prompt-chunk rows k_new/v_new
    [T][Hkv][D] at the last q_len_b positions of each request (q_offsets [B+1]
    int32 cuda); with inv_freq, q [T][Hq][D] and k are RoPE-rotated first."""
    import torch
    for name, t in (("k_pages", k_pages), ("v_pages", v_pages), ("block_table", block_table), ("seq_lens", seq_lens),
                    ("q_offsets", q_offsets), ("k_new", k_new), ("v_new", v_new)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if q_offsets.dtype != torch.int32 or not q_offsets.is_contiguous():
        raise ValueError("q_offsets must be contiguous int32")
    if k_new.dtype != torch.bfloat16 or not k_new.is_contiguous() or not v_new.is_contiguous():
        raise ValueError("k_new / v_new must be contiguous bf16")
    if inv_freq is not None and (q is None or not q.is_cuda or not q.is_contiguous() or inv_freq.dtype != torch.float32):
        raise ValueError("RoPE needs a contiguous cuda q and a float32 inv_freq")
    npages, hkv, P, d = k_pages.shape
    check(lib().neo_prefill_append(q.data_ptr() if q is not None else None, q.shape[1] if q is not None else 0,
                                   inv_freq.data_ptr() if inv_freq is not None else None, k_pages.data_ptr(),
                                   v_pages.data_ptr(), k_pages.stride(0),
                                   int(num_pages if num_pages is not None else npages), block_table.data_ptr(),
                                   block_table.shape[1], seq_lens.data_ptr(), q_offsets.data_ptr(), k_new.data_ptr(),
                                   v_new.data_ptr(), seq_lens.shape[0], k_new.shape[0], hkv, d, P, _stream(stream)))


# ------------------------------------------------------------------ scheduler


class CostModel(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("t_pre_layer_s", ctypes.c_double),
                ("t_post_layer_s", ctypes.c_double), ("lin_tokens", ctypes.c_void_p), ("lin_s", ctypes.c_void_p),
                ("lin_n", ctypes.c_int32), ("gdec_tokens", ctypes.c_void_p), ("gdec_s", ctypes.c_void_p),
                ("gdec_n", ctypes.c_int32), ("gpre_a", ctypes.c_double), ("gpre_b", ctypes.c_double),
                ("cdec_tokens", ctypes.c_void_p), ("cdec_s", ctypes.c_void_p), ("cdec_n", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("max_batch_tokens", ctypes.c_int64),
                ("pcie_bytes_per_s", ctypes.c_double), ("kv_bytes_per_token_layer", ctypes.c_double)]


class SchedPlan(ctypes.Structure):
    _fields_ = [("two_batch", ctypes.c_int32), ("x", ctypes.c_int32), ("n_batch0", ctypes.c_int32),
                ("n_batch1", ctypes.c_int32), ("n_swap_out", ctypes.c_int32), ("n_swap_in", ctypes.c_int32),
                ("t_iter", ctypes.c_double), ("t_l0", ctypes.c_double), ("t_l1", ctypes.c_double),
                ("t_ga0", ctypes.c_double), ("t_ca0", ctypes.c_double), ("t_ca1", ctypes.c_double)]


class SchedRequest(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int64), ("kind", ctypes.c_int32), ("ctx", ctypes.c_int32)]


def schedule(profile: dict, reqs, gpu_free_pages: int, cpu_free_pages: int) -> dict:
    """neo_schedule.  profile: L, t_prl, t_pol, lin/gdec/cdec tables
    [(tokens, s)], gpre_a, gpre_b, page_size, max_batch_tokens, pcie_bytes_per_s,
    kv_bytes_per_token_layer.  reqs: [(id, kind, ctx)] in queue order (kind 0 =
    waiting, 1 = GPU decoding, 2 = CPU decoding)."""
    tabs = {}
    for name in ("lin", "gdec", "cdec"):
        t = np.ascontiguousarray(np.asarray(profile[name], dtype=np.float64).reshape(-1, 2).T)
        tabs[name] = (np.ascontiguousarray(t[0]), np.ascontiguousarray(t[1]))
    m = CostModel(int(profile["L"]), float(profile["t_prl"]), float(profile["t_pol"]),
                  tabs["lin"][0].ctypes.data, tabs["lin"][1].ctypes.data, len(tabs["lin"][0]),
                  tabs["gdec"][0].ctypes.data, tabs["gdec"][1].ctypes.data, len(tabs["gdec"][0]),
                  float(profile["gpre_a"]), float(profile["gpre_b"]),
                  tabs["cdec"][0].ctypes.data, tabs["cdec"][1].ctypes.data, len(tabs["cdec"][0]),
                  int(profile["page_size"]), int(profile["max_batch_tokens"]),
                  float(profile["pcie_bytes_per_s"]), float(profile["kv_bytes_per_token_layer"]))
    n = len(reqs)
    arr = (SchedRequest * max(n, 1))(*[SchedRequest(int(i), int(k), int(c)) for i, k, c in reqs])
    outs = [np.zeros(max(n, 1), dtype=np.int64) for _ in range(4)]
    plan = SchedPlan()
    check(lib().neo_schedule(ctypes.byref(m), arr, n, int(gpu_free_pages), int(cpu_free_pages),
                             *[o.ctypes.data for o in outs], ctypes.byref(plan)))
    return {"two_batch": bool(plan.two_batch), "x": plan.x, "batch0": outs[0][:plan.n_batch0].tolist(),
            "batch1": outs[1][:plan.n_batch1].tolist(), "swap_out": outs[2][:plan.n_swap_out].tolist(),
            "swap_in": outs[3][:plan.n_swap_in].tolist(), "t_iter": plan.t_iter, "t_l0": plan.t_l0,
            "t_l1": plan.t_l1, "t_ga0": plan.t_ga0, "t_ca0": plan.t_ca0, "t_ca1": plan.t_ca1}


# ------------------------------------------------------------------ KV pool


class KVPool:
    """GPU-cache + CPU-cache pool.  The device pool and the pinned
    host pool are torch tensors owned by this object; the C handle owns only the
    free lists."""

    def __init__(self, num_layers: int, num_kv_heads: int, num_gpu_pages: int, num_host_pages: int = 0,
                 page_size: int = 16, head_dim: int = 128, device=None, allocate: bool = True,
                 gpu_buffer=None, host_buffer=None, host_array=None):
        """gpu_buffer/host_buffer: optional caller-owned tensors (bf16, at least
        gpu_bytes/host_bytes, host one pinned) to wrap instead of allocating."""
        self.geo = Geometry(num_layers, num_kv_heads, head_dim, page_size, num_gpu_pages, num_host_pages)
        gb, hb = ctypes.c_size_t(), ctypes.c_size_t()
        check(lib().neo_kv_pool_bytes(ctypes.byref(self.geo), ctypes.byref(gb), ctypes.byref(hb)))
        self.gpu_bytes, self.host_bytes = gb.value, hb.value
        self.gpu = self.host = None
        # allocate=False: accounting-only handle (allocator tests); sentinel bases
        # that are never dereferenced because no swap/attention runs on it.
        gptr, hptr = (1 << 40), ((1 << 41) if num_host_pages else None)
        self.host_array = None
        if not allocate and host_array is not None:
            # CPU-only pool (CPU attention tests): a numpy uint16 CPU-cache
            if host_array.dtype != np.uint16 or host_array.nbytes < self.host_bytes:
                raise ValueError("host_array must be uint16 and hold host_bytes")
            self.host_array = host_array
            hptr = host_array.ctypes.data
        if allocate:
            import torch
            if gpu_buffer is not None:
                if gpu_buffer.numel() * gpu_buffer.element_size() < self.gpu_bytes or not gpu_buffer.is_cuda:
                    raise ValueError("gpu_buffer too small or not on CUDA")
                self.gpu = gpu_buffer.reshape(-1).view(torch.bfloat16)[: self.gpu_bytes // 2]
            else:
                self.gpu = torch.empty(self.gpu_bytes // 2, dtype=torch.bfloat16, device=device or "cuda")
            gptr = self.gpu.data_ptr()
            if num_host_pages:
                if host_buffer is not None:
                    if host_buffer.numel() * host_buffer.element_size() < self.host_bytes or not host_buffer.is_pinned():
                        raise ValueError("host_buffer too small or not pinned")
                    self.host = host_buffer.reshape(-1).view(torch.bfloat16)[: self.host_bytes // 2]
                else:
                    self.host = torch.empty(self.host_bytes // 2, dtype=torch.bfloat16, pin_memory=True)
                hptr = self.host.data_ptr()
        self._h = ctypes.c_void_p()
        check(lib().neo_kv_pool_create(ctypes.byref(self.geo), gptr, self.gpu_bytes, hptr, self.host_bytes,
                                       ctypes.byref(self._h)))

    def close(self):
        if self._h:
            lib().neo_kv_pool_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def alloc(self, where: int, n: int) -> np.ndarray:
        ids = np.zeros(max(n, 1), dtype=np.int32)
        check(lib().neo_kv_alloc(self._h, where, n, ids.ctypes.data))
        return ids[:n].copy()

    def free(self, where: int, ids) -> None:
        a = _ids(ids)
        check(lib().neo_kv_free(self._h, where, len(a), a.ctypes.data))

    def free_count(self, where: int) -> int:
        n = ctypes.c_int64()
        check(lib().neo_kv_free_count(self._h, where, ctypes.byref(n)))
        return n.value

    def gpu_view(self):
        """[L][2][num_gpu_pages][Hkv][P][D] view of the GPU-cache."""
        g = self.geo
        return self.gpu.view(g.num_layers, 2, g.num_gpu_pages, g.num_kv_heads, g.page_size, g.head_dim)

    def host_view(self):
        """[num_host_pages][L][2][Hkv][P][D] view of the CPU-cache."""
        g = self.geo
        return self.host.view(g.num_host_pages, g.num_layers, 2, g.num_kv_heads, g.page_size, g.head_dim)

    def layer_view(self, layer: int):
        """(k_pages, v_pages) [num_gpu_pages][Hkv][P][D] torch views via neo_kv_layer_view."""
        import torch
        k, v, stride = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        check(lib().neo_kv_layer_view(self._h, layer, ctypes.byref(k), ctypes.byref(v), ctypes.byref(stride)))
        g = self.geo
        base = self.gpu.data_ptr()
        ko = (k.value - base) // 2
        vo = (v.value - base) // 2
        shape = (g.num_gpu_pages, g.num_kv_heads, g.page_size, g.head_dim)
        strides = (stride.value, g.page_size * g.head_dim, g.head_dim, 1)
        return (torch.as_strided(self.gpu, shape, strides, ko), torch.as_strided(self.gpu, shape, strides, vo))

    def cpu_decode_attn(self, layer: int, q, host_block_table, seq_lens, out=None, scale=None,
                        num_threads: int = 0):
        """neo_cpu_decode_attn (NEXT-2): host q [B][Hq][D] bf16 bits
        (numpy uint16 or a CPU torch bf16 tensor), host table/seq_lens -> out."""
        qa = _host_u16(q)
        B, hq, d = qa.shape
        tab = np.ascontiguousarray(np.asarray(host_block_table, dtype=np.int32))
        sl = np.ascontiguousarray(np.asarray(seq_lens, dtype=np.int32))
        o = np.empty_like(qa) if out is None else out
        check(lib().neo_cpu_decode_attn(self._h, layer, qa.ctypes.data, tab.ctypes.data, tab.shape[1], sl.ctypes.data,
                                        o.ctypes.data, B, hq, float(scale if scale is not None else 1 / math.sqrt(d)),
                                        num_threads))
        return o

    def staging_bytes(self, n: int, layer_begin: int = 0, layer_end: int | None = None) -> int:
        le = self.geo.num_layers if layer_end is None else layer_end
        out = ctypes.c_size_t()
        check(lib().neo_kv_swap_staging_bytes(self._h, n, layer_begin, le, ctypes.byref(out)))
        return out.value

    def swap_out(self, gpu_ids, host_ids, staging, layer_begin: int = 0, layer_end: int | None = None,
                 stream=None, defer_join: bool = False) -> None:
        """neo_kv_swap_out (defer_join: neo_kv_swap_out_ex with NEO_SWAP_DEFER_JOIN);
        staging=None selects the zero-copy path."""
        g, h = _ids(gpu_ids), _ids(host_ids)
        if len(g) != len(h):
            raise ValueError("gpu_ids and host_ids differ in length")
        le = self.geo.num_layers if layer_end is None else layer_end
        nbytes = 0 if staging is None else staging.numel() * staging.element_size()
        if defer_join:
            check(lib().neo_kv_swap_out_ex(self._h, len(g), g.ctypes.data, h.ctypes.data, layer_begin, le,
                                           _ptr(staging), nbytes, NEO_SWAP_DEFER_JOIN, _stream(stream)))
        else:
            check(lib().neo_kv_swap_out(self._h, len(g), g.ctypes.data, h.ctypes.data, layer_begin, le,
                                        _ptr(staging), nbytes, _stream(stream)))

    def swap_join(self, stream=None) -> None:
        """neo_kv_swap_join: `stream` waits for every PCIe copy of this pool's swaps so far."""
        check(lib().neo_kv_swap_join(self._h, _stream(stream)))

    def swap_in(self, host_ids, gpu_ids, staging, layer_begin: int = 0, layer_end: int | None = None,
                stream=None) -> None:
        g, h = _ids(gpu_ids), _ids(host_ids)
        if len(g) != len(h):
            raise ValueError("gpu_ids and host_ids differ in length")
        le = self.geo.num_layers if layer_end is None else layer_end
        nbytes = 0 if staging is None else staging.numel() * staging.element_size()
        check(lib().neo_kv_swap_in(self._h, len(g), h.ctypes.data, g.ctypes.data, layer_begin, le,
                                   _ptr(staging), nbytes, _stream(stream)))
