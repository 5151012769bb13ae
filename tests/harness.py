"""Test harness: builds paged GPU inputs and their unpaged oracle counterparts
from the same seeded generator (neo_inputs), and the tolerance rule.

The oracle always receives K/V straight from the generator (unpaged, per
request), never from the paged pool the GPU reads, so a paging or
block-table bug cannot cancel out."""
from __future__ import annotations

import math

import numpy as np

import neo_inputs as ni

ATOL, RTOL = 2e-3, 1e-2          # north_star: max |err| <= 2e-3 abs + 1e-2 rel
D = 128
NAN_BF16 = 0x7FC0


def within_tol(gpu: np.ndarray, ref: np.ndarray):
    err = np.abs(gpu - ref)
    lim = ATOL + RTOL * np.abs(ref)
    ratio = float(np.max(err / lim)) if err.size else 0.0
    return bool(np.all(err <= lim) and np.all(np.isfinite(gpu))), ratio


class Case:
    """A batch of requests: host bit arrays + device tensors."""

    def __init__(self, ctx, hq, hkv, P=16, seed=0x4E454F, layer=0, variant=0, extra_pages=3, tail="nan",
                 page_stride=None, table_seed=None, b_offset=0, fill_unused="nan"):
        import torch
        self.ctx = np.asarray(ctx, dtype=np.int32)
        self.B, self.hq, self.hkv, self.P = len(self.ctx), hq, hkv, P
        self.seed, self.layer, self.variant, self.b_offset = seed, layer, variant, b_offset
        need = int(ni.pages_needed(self.ctx, P).sum())
        self.table, self.npages = ni.block_tables(seed if table_seed is None else table_seed, self.ctx, P,
                                                  num_pages=need + extra_pages)
        self.max_blocks = self.table.shape[1]
        self.max_seq_len = max(int(self.ctx.max()) if self.B else 0, 1)
        fill = NAN_BF16 if fill_unused == "nan" else 0
        kp = np.full((self.npages, hkv, P, D), fill, dtype=np.uint16)
        vp = np.full((self.npages, hkv, P, D), fill, dtype=np.uint16)
        self.q = ni.q_bits(seed, layer, np.arange(self.B) + b_offset, hq, D, variant=variant)
        self.k_req, self.v_req = [], []
        for b in range(self.B):
            n = int(self.ctx[b])
            kb = ni.kv_bits(seed, layer, ni.KIND_K, b + b_offset, 0, n, hkv, D, variant=variant, hq_total=hq)
            vb = ni.kv_bits(seed, layer, ni.KIND_V, b + b_offset, 0, n, hkv, D)
            self.k_req.append(kb)
            self.v_req.append(vb)
            npg = (n + P - 1) // P
            for j in range(npg):
                pid = self.table[b, j]
                t0, t1 = j * P, min(n, (j + 1) * P)
                kp[pid, :, :t1 - t0] = kb[t0:t1].transpose(1, 0, 2)
                vp[pid, :, :t1 - t0] = vb[t0:t1].transpose(1, 0, 2)
                if t1 - t0 < P and tail != "nan":
                    tv = 0 if tail == "zero" else fill
                    kp[pid, :, t1 - t0:] = tv
                    vp[pid, :, t1 - t0:] = tv
        self.kpool, self.vpool = kp, vp
        # device tensors; optional padded page stride (page-major style layouts)
        stride = hkv * P * D if page_stride is None else page_stride
        self.page_stride = stride

        def dev_pool(host):
            buf = torch.full((self.npages * stride + 64,), float("nan"), dtype=torch.bfloat16, device="cuda")
            view = torch.as_strided(buf, (self.npages, hkv, P, D), (stride, P * D, D, 1))
            view.copy_(torch.from_numpy(host.view(np.int16)).cuda().view(torch.bfloat16))
            return buf, view

        self._kbuf, self.k_dev = dev_pool(kp)
        self._vbuf, self.v_dev = dev_pool(vp)
        self.q_dev = torch.from_numpy(self.q.view(np.int16)).cuda().view(torch.bfloat16)
        self.bt_dev = torch.from_numpy(self.table).cuda()
        self.sl_dev = torch.from_numpy(self.ctx).cuda()
        self.scale = 1.0 / math.sqrt(D)

    def run(self, chunk_tokens=0, out=None, workspace=None, block_table=None):
        from paper_2411_01142_b200 import neo
        import torch
        o = neo.decode_attn(self.q_dev, self.k_dev, self.v_dev, self.bt_dev if block_table is None else block_table,
                            self.sl_dev, self.max_seq_len, chunk_tokens=chunk_tokens, out=out, workspace=workspace,
                            scale=self.scale)
        torch.cuda.synchronize()
        return o

    def out_f64(self, out):
        import torch
        return ni.bf16_bits_to_f64(out.view(torch.int16).cpu().numpy().view(np.uint16))

    def oracle(self, b):
        import oracle
        return oracle.decode_attention(self.q[b], self.k_req[b], self.v_req[b], np.float32(self.scale))


class PrefillCase(Case):
    """Prompt chunks: request b's last q_lens[b] tokens (of ctx[b]) are the query
    rows, packed as q [T][Hq][D] with offsets q_off [B+1]; the pool already holds
    all ctx[b] tokens (as neo_prefill_append leaves it)."""

    def __init__(self, ctx, q_lens, hq, hkv, **kw):
        import torch
        super().__init__(ctx, hq, hkv, **kw)
        self.q_lens = np.asarray(q_lens, dtype=np.int32)
        assert np.all(self.q_lens <= self.ctx) and np.all(self.q_lens >= 0)
        self.q_off = np.zeros(self.B + 1, dtype=np.int32)
        self.q_off[1:] = np.cumsum(self.q_lens)
        self.T = int(self.q_off[-1])
        self.max_q_len = max(int(self.q_lens.max()) if self.B else 0, 1)
        # per-token q rows: global token ids offset so they never collide with decode q rows
        self.qp = ni.q_bits(self.seed, self.layer, np.arange(self.T) + 1_000_000 + 4096 * self.b_offset, hq, D,
                            variant=self.variant)
        self.qp_dev = torch.from_numpy(self.qp.view(np.int16)).cuda().view(torch.bfloat16)
        self.qo_dev = torch.from_numpy(self.q_off).cuda()

    def run(self, out=None, scale=None):
        from paper_2411_01142_b200 import neo
        import torch
        o = neo.prefill_attn(self.qp_dev, self.k_dev, self.v_dev, self.bt_dev, self.sl_dev, self.qo_dev,
                             self.max_q_len, out=out, scale=self.scale if scale is None else scale)
        torch.cuda.synchronize()
        return o

    def rows(self, b):
        return slice(int(self.q_off[b]), int(self.q_off[b + 1]))

    def oracle(self, b):
        import oracle
        return oracle.prefill_attention(self.qp[self.rows(b)], self.k_req[b], self.v_req[b], np.float32(self.scale))
