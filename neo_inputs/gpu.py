"""Materialise a workload's synthetic inputs in HBM with the device generator:
a layer-major KV pool [L][2][num_pages][Hkv][P][D] (the layout of include/neo.h),
per-layer q, a scattered block table and seq_lens.  Input construction only."""
from __future__ import annotations

import numpy as np

import neo_inputs as ni
from neo_inputs import device as gen


class GpuBatch:
    def __init__(self, wl, ctx=None, layers=None, kv_heads=None, q_heads=None, req_ids=None, device="cuda",
                 variant=0, extra_pages=0, tail=gen.TAIL_NAN):
        """kv_heads/q_heads: (begin, end) global head ranges of this rank's shard;
        req_ids: global request ids of this rank's share (default: all)."""
        import torch
        self.wl = wl
        full_ctx = wl.contexts() if ctx is None else np.asarray(ctx, dtype=np.int32)
        self.req_ids = np.arange(len(full_ctx)) if req_ids is None else np.asarray(req_ids)
        self.ctx = full_ctx[self.req_ids].astype(np.int32)
        self.layers = wl.layers_built if layers is None else layers
        self.kv_heads = (0, wl.hkv) if kv_heads is None else kv_heads
        self.q_heads = (0, wl.hq) if q_heads is None else q_heads
        self.hkv = self.kv_heads[1] - self.kv_heads[0]
        self.hq = self.q_heads[1] - self.q_heads[0]
        self.B = len(self.ctx)
        P = self.P = wl.page_size
        need = ni.pages_needed(self.ctx, P)
        self.num_pages = int(need.sum()) + extra_pages
        self.table, _ = ni.block_tables(wl.seed, self.ctx, P, num_pages=self.num_pages)
        self.max_blocks = self.table.shape[1]
        self.max_seq_len = int(self.ctx.max()) if self.B else 1
        self.variant = variant
        pe = self.hkv * P * 128
        self.pool = torch.empty((self.layers, 2, self.num_pages, self.hkv, P, 128), dtype=torch.bfloat16,
                                device=device)
        self.q = torch.empty((self.layers, self.B, self.hq, 128), dtype=torch.bfloat16, device=device)
        self.block_table = torch.from_numpy(self.table).to(device)
        self.seq_lens = torch.from_numpy(self.ctx).to(device)
        # contiguous request runs share a b_offset; fill per run of consecutive ids
        runs = _runs(self.req_ids)
        for layer in range(self.layers):
            k, v = self.pool[layer, 0], self.pool[layer, 1]
            for lo, hi, gid in runs:
                gen.fill_kv(k, v, self.block_table[lo:hi], self.seq_lens[lo:hi], seed=wl.seed, layer=layer,
                            hkv_total=wl.hkv, g_offset=self.kv_heads[0], hq_total=wl.hq, b_offset=gid,
                            variant=variant, tail=tail)
                gen.fill_q(self.q[layer, lo:hi], seed=wl.seed, layer=layer, hq_total=wl.hq,
                           h_offset=self.q_heads[0], b_offset=gid, variant=variant)
        self.page_elems = pe

    def layer(self, layer: int):
        return self.pool[layer % self.layers, 0], self.pool[layer % self.layers, 1]

    def kv_bytes_per_call(self) -> int:
        return int(self.ctx.astype(np.int64).sum()) * self.hkv * 128 * 2 * 2

    def other_bytes_per_call(self) -> int:
        n_pages = int(ni.pages_needed(self.ctx, self.P).sum())
        return 2 * self.B * self.hq * 128 * 2 + 4 * n_pages + 4 * self.B

    # host-side oracle inputs for one request of this batch (global ids)
    def oracle_inputs(self, b_local: int, layer: int):
        gid = int(self.req_ids[b_local])
        n = int(self.ctx[b_local])
        heads = np.arange(*self.kv_heads)
        qh = np.arange(*self.q_heads)
        q = ni.q_bits(self.wl.seed, layer, [gid], self.wl.hq, 128, heads=qh, variant=self.variant)[0]
        k = ni.kv_bits(self.wl.seed, layer, ni.KIND_K, gid, 0, n, self.wl.hkv, 128, heads=heads,
                       variant=self.variant, hq_total=self.wl.hq)
        v = ni.kv_bits(self.wl.seed, layer, ni.KIND_V, gid, 0, n, self.wl.hkv, 128, heads=heads)
        return q, k, v


def _runs(ids):
    """[(lo, hi, global_id_of_lo)] runs of consecutive global ids."""
    out = []
    lo = 0
    for i in range(1, len(ids) + 1):
        if i == len(ids) or ids[i] != ids[i - 1] + 1:
            out.append((lo, i, int(ids[lo])))
            lo = i
    return out
