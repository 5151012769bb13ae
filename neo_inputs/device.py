"""Device side of the seeded input generator (libneo_gen.so, csrc/neo_gen.cu).

Writes the same bit patterns as ``neo_inputs`` (host) straight into GPU
buffers, so full-size workloads (tens of GB of KV) are built in HBM.  Contains
no attention arithmetic."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libneo_gen.so")
_lib = None

TAIL_VALUES, TAIL_NAN, TAIL_ZERO = 0, 1, 2


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} not built: run `python -m paper_2411_01142_b200.build`")
        L = ctypes.CDLL(_LIB)
        P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.neo_gen_fill_kv.argtypes = [P, P, i64, P, i32, P, i32, i32, i32, i32, i32, i32, i32, i32, u64, i32, i32,
                                      i32, P]
        L.neo_gen_fill_q.argtypes = [P, i32, i32, i32, i32, i32, i32, u64, i32, i32, P]
        L.neo_gen_values.argtypes = [u64, ctypes.c_uint32, P, i64, P, P]
        for f in (L.neo_gen_fill_kv, L.neo_gen_fill_q, L.neo_gen_values):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _stream(stream):
    import torch
    s = stream or torch.cuda.current_stream()
    return s.cuda_stream


def _ok(rc):
    if rc != 0:
        raise RuntimeError(f"neo_gen CUDA error {rc}")


def fill_kv(k_pages, v_pages, block_table, seq_lens, *, seed, layer, hkv_total=None, g_offset=0, hq_total,
            b_offset=0, variant=0, tail=TAIL_VALUES, stream=None):
    """Fill the pages referenced by ``block_table``/``seq_lens`` of one layer.
    k_pages/v_pages: [num_pages][Hkv_local][P][D] bf16 views (page stride = stride(0))."""
    npages, hkv, P, d = k_pages.shape
    B, max_blocks = block_table.shape
    _ok(lib().neo_gen_fill_kv(k_pages.data_ptr(), v_pages.data_ptr(), k_pages.stride(0), block_table.data_ptr(),
                              max_blocks, seq_lens.data_ptr(), B, b_offset, hkv, g_offset,
                              hkv_total if hkv_total is not None else hkv, hq_total, d, P, seed, layer, variant,
                              tail, _stream(stream)))


def fill_q(q, *, seed, layer, hq_total=None, h_offset=0, b_offset=0, variant=0, stream=None):
    B, hq, d = q.shape
    _ok(lib().neo_gen_fill_q(q.data_ptr(), B, b_offset, hq, h_offset, hq_total if hq_total is not None else hq, d,
                             seed, layer, variant, _stream(stream)))


def values(seed: int, tid: int, idx: np.ndarray):
    """bf16 bits for indices ``idx`` computed on the device (for the host/device
    bit-equality test)."""
    import torch
    t_idx = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.uint64).view(np.int64)).cuda()
    out = torch.empty(len(idx), dtype=torch.int16, device="cuda")
    _ok(lib().neo_gen_values(seed, tid, t_idx.data_ptr(), len(idx), out.data_ptr(), _stream(None)))
    return out.cpu().numpy().view(np.uint16)
