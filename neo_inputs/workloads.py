"""BASELINE.json's five configurations as synthetic workload recipes
(SURVEY §8(d) table).  Shapes are LLaMa's; values come from the counter-based
generator; context lengths follow the paper's synthetic recipe or the
config text.  No attention arithmetic here."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import neo_inputs as ni

BASE_SEED = ni.DEFAULT_SEED


@dataclass(frozen=True)
class Workload:
    name: str
    model: str
    hq: int
    hkv: int
    batch: int
    num_layers: int          # layers of the model (KV materialised for layers_built)
    layers_built: int        # distinct layer pools kept in HBM and cycled through
    ctx_kind: str
    ctx_args: tuple
    page_size: int = 16
    swap_requests: int = 0   # requests swapped out to pinned host concurrently (c3)
    note: str = ""
    index: int = 0

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index

    def contexts(self) -> np.ndarray:
        k, a = self.ctx_kind, self.ctx_args
        if k == "fixed":
            return np.full(self.batch, a[0], dtype=np.int32)
        if k == "uniform":       # U_int[ceil(0.9 l), floor(1.1 l)]
            return ni.ctx_uniform(self.seed, self.batch, a[0])
        if k == "range":
            return ni.ctx_range(self.seed, self.batch, a[0], a[1])
        if k == "loguniform":
            return ni.ctx_loguniform(self.seed, self.batch, a[0], a[1])
        if k == "lognormal":
            return ni.ctx_lognormal(self.seed, self.batch, *a)
        raise ValueError(k)

    def kv_bytes_per_token_layer(self) -> int:
        return self.hkv * 128 * 2 * 2


WORKLOADS = {
    "c1": Workload("c1", "LLaMa-2-7B", 32, 32, 4, 32, 1, "fixed", (128,), index=1,
                   note="single layer, MHA, batch 4, ctx 128 (latency config)"),
    "c2": Workload("c2", "LLaMa-3.1-8B", 32, 8, 256, 32, 32, "uniform", (1024,), index=2,
                   note="all 32 layers, batch 256, ctx ~U_int[922,1126] (code-generation-like)"),
    "c2s": Workload("c2s", "LLaMa-3.1-8B", 32, 8, 256, 32, 32, "lognormal", (1024, 0.75, 16, 8192), index=2,
                    note="skewed variant: lognormal median 1K, sigma 0.75, clip [16, 8192] (P:410)"),
    "c3": Workload("c3", "LLaMa-3.1-8B", 32, 8, 128, 32, 32, "range", (4096, 8192), swap_requests=16, index=3,
                   note="batch 128, ctx U_int[4096,8192] (summarization-like), 16 requests swapped out"),
    "c4": Workload("c4", "LLaMa-3.1-70B", 64, 8, 512, 80, 4, "uniform", (2048,), index=4,
                   note="batch 512, ctx ~U_int[1844,2252], 4 distinct layer pools cycled (80 layers do not fit)"),
    "c5": Workload("c5", "LLaMa-3.1-8B", 32, 8, 1024, 32, 1, "loguniform", (128, 16384), index=5,
                   note="1024 requests, ctx floor(exp(U[ln128, ln16384])), GPU-resident fraction f"),
}

