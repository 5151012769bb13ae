"""oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain, slow, obviously-correct references for NEO's GPU hot path.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA library; the CUDA path never imports it.

* ``decode_attention`` / ``decode_attention_batch`` / ``softmax_weights`` /
  ``partial`` / ``merge`` -- fp64 C (``neo_oracle.c``), unpaged K/V; cites
  P:97-98, P:109-110, P:122, P:307 and S:451, S:468-471 (see the C header).
* ``prefill_attention`` -- causal prefill (P:237-239 prefill in batch-0; row i
  of the prompt chunk sees the tokens up to its own position), the decode
  definition applied row by row.
* ``gather_pages`` / ``host_record`` -- the page-swap definition (P:235
  "entirely in the GPU-cache ... or entirely in the CPU-cache", P:240
  layer-wise swapping, P:285-288 swap-out/in): a bit copy of the request's pages
  for a layer range, written as numpy indexing.

Pinned against closed forms, brute force and invariants in
``tests/test_oracle_pins.py`` (the batch driver against fp64 torch SDPA and
bitwise against the single-request call; the softmax weights against fp64
torch.softmax and Decimal brute force).  Every exported function is pinned
(DESIGN.md §3).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "neo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            lib.oracle_decode_attention.argtypes = [P, P, P, i64, i32, i32, i32, f64, P]
            lib.oracle_softmax_weights.argtypes = [P, P, i64, i32, i32, i32, f64, P]
            lib.oracle_partial.argtypes = [P, P, P, i32, i32, i32, i32, i64, i64, f64, P, P, P]
            lib.oracle_merge.argtypes = [i32, P, P, P, i32, P]
            lib.oracle_decode_attention_batch.argtypes = [P, P, P, P, i64, i32, i32, i32, f64, P, i32]
            lib.oracle_prefill_attention.argtypes = [P, P, P, i64, i64, i32, i32, i32, f64, P, i32]
            for f in (lib.oracle_decode_attention, lib.oracle_softmax_weights, lib.oracle_partial,
                      lib.oracle_merge, lib.oracle_decode_attention_batch, lib.oracle_prefill_attention):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _u16(a):
    a = np.ascontiguousarray(a, dtype=np.uint16)
    return a, a.ctypes.data


def decode_attention(q_bits, k_bits, v_bits, scale: float) -> np.ndarray:
    """One request. q_bits [Hq][D], k_bits/v_bits [n][Hkv][D] (bf16 bits) ->
    out [Hq][D] float64."""
    q, qp = _u16(q_bits)
    k, kp = _u16(k_bits)
    v, vp = _u16(v_bits)
    hq, d = q.shape
    n, hkv, d2 = k.shape if k.ndim == 3 else (0, 1, d)
    out = np.zeros((hq, d), dtype=np.float64)
    rc = _load().oracle_decode_attention(qp, kp, vp, n, hq, hkv, d, float(scale), out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_decode_attention rc={rc}")
    return out


def softmax_weights(q_bits, k_bits, scale: float) -> np.ndarray:
    q, qp = _u16(q_bits)
    k, kp = _u16(k_bits)
    hq, d = q.shape
    n, hkv, _ = k.shape
    w = np.zeros((hq, n), dtype=np.float64)
    rc = _load().oracle_softmax_weights(qp, kp, n, hq, hkv, d, float(scale), w.ctypes.data)
    if rc:
        raise ValueError(f"oracle_softmax_weights rc={rc}")
    return w


def partial(q_bits, k_bits, v_bits, h: int, t0: int, t1: int, scale: float):
    """(m, l, acc[D]) of one flash-decoding task for q-head h over [t0, t1)."""
    q, qp = _u16(q_bits)
    k, kp = _u16(k_bits)
    v, vp = _u16(v_bits)
    hq, d = q.shape
    hkv = k.shape[1]
    m = ctypes.c_double()
    l = ctypes.c_double()
    acc = np.zeros(d, dtype=np.float64)
    rc = _load().oracle_partial(qp, kp, vp, hq, hkv, d, h, t0, t1, float(scale), ctypes.byref(m),
                                ctypes.byref(l), acc.ctypes.data)
    if rc:
        raise ValueError(f"oracle_partial rc={rc}")
    return m.value, l.value, acc


def merge(ms, ls, accs) -> np.ndarray:
    m = np.ascontiguousarray(ms, dtype=np.float64)
    l = np.ascontiguousarray(ls, dtype=np.float64)
    a = np.ascontiguousarray(accs, dtype=np.float64)
    d = a.shape[1]
    out = np.zeros(d, dtype=np.float64)
    rc = _load().oracle_merge(len(m), m.ctypes.data, l.ctypes.data, a.ctypes.data, d, out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_merge rc={rc}")
    return out


def decode_attention_batch(q_bits, k_list, v_list, scale: float, nthreads: int = 1) -> np.ndarray:
    """q_bits [B][Hq][D]; k_list/v_list: per-request [n_b][Hkv][D]. Threads over
    requests (used for the cpu_baseline timing)."""
    q, qp = _u16(q_bits)
    B, hq, d = q.shape
    hkv = k_list[0].shape[1]
    lens = np.array([x.shape[0] for x in k_list], dtype=np.int64)
    offsets = np.zeros(B + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(lens)
    k = np.ascontiguousarray(np.concatenate(k_list, axis=0), dtype=np.uint16)
    v = np.ascontiguousarray(np.concatenate(v_list, axis=0), dtype=np.uint16)
    out = np.zeros((B, hq, d), dtype=np.float64)
    rc = _load().oracle_decode_attention_batch(qp, k.ctypes.data, v.ctypes.data, offsets.ctypes.data,
                                               B, hq, hkv, d, float(scale), out.ctypes.data,
                                               int(nthreads))
    if rc:
        raise ValueError(f"oracle_decode_attention_batch rc={rc}")
    return out


def prefill_attention(q_bits, k_bits, v_bits, scale: float, nthreads: int = 0) -> np.ndarray:
    """Causal prefill of one request (neo_oracle.c ``oracle_prefill_attention``).
    q_bits [n_q][Hq][D]: the last n_q of the n tokens in k_bits/v_bits [n][Hkv][D];
    row i attends to tokens 0 .. n - n_q + i.  Returns [n_q][Hq][D] float64."""
    q, qp = _u16(q_bits)
    k, kp = _u16(k_bits)
    v, vp = _u16(v_bits)
    n_q, hq, d = q.shape
    n, hkv, _ = k.shape
    out = np.zeros((n_q, hq, d), dtype=np.float64)
    nth = nthreads or min(32, os.cpu_count() or 1)
    rc = _load().oracle_prefill_attention(qp, kp, vp, n, n_q, hq, hkv, d, float(scale), out.ctypes.data, nth)
    if rc:
        raise ValueError(f"oracle_prefill_attention rc={rc}")
    return out


# ------------------------------------------------------------------ page swap


def gather_pages(gpu_pool: np.ndarray, gpu_ids, layer_begin: int, layer_end: int) -> np.ndarray:
    """Swap-out record of a request: ``gpu_pool`` is the GPU-cache
    ``[L][2][num_pages][Hkv][P][D]``; returns ``[n][layer_end-layer_begin][2][Hkv][P][D]``
    holding the same bits, page by page in the order given."""
    ids = np.asarray(gpu_ids, dtype=np.int64)
    sub = gpu_pool[layer_begin:layer_end][:, :, ids]          # [Lr][2][n][Hkv][P][D]
    return np.ascontiguousarray(np.moveaxis(sub, 2, 0))


def host_record(host_pool: np.ndarray, host_ids, layer_begin: int, layer_end: int) -> np.ndarray:
    """The layer slice of CPU-cache pages ``host_pool[num_host][L][2][Hkv][P][D]``."""
    ids = np.asarray(host_ids, dtype=np.int64)
    return np.ascontiguousarray(host_pool[ids][:, layer_begin:layer_end])
