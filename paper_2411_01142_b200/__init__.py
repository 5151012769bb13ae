"""NEO (arXiv 2411.01142) hot path on B200: paged GQA decode attention over a
GPU-cache plus the KV page swap to/from a pinned CPU-cache, as a C-ABI CUDA
library (include/neo.h, libneo.so) with a thin Python binding (neo.py)."""
from .neo import (NEO_GPU, NEO_HOST, KVPool, NeoError, decode_attn, default_chunk, lib, make_workspace,
                  workspace_bytes)

__all__ = ["NEO_GPU", "NEO_HOST", "KVPool", "NeoError", "decode_attn", "default_chunk", "lib", "make_workspace",
           "workspace_bytes"]
