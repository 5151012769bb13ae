"""oracle/rope.py -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Rotary position embedding (RoFormer, rotate-half convention as used by LLaMa),
the operation neo_rope_append fuses into the KV append, written
from its definition in fp64: for position t and dim pair (i, i + D/2),
theta_i = t * inv_freq[i],
    x'[i]       = x[i] cos theta_i - x[i + D/2] sin theta_i
    x'[i + D/2] = x[i + D/2] cos theta_i + x[i] sin theta_i
Pinned in tests/test_oracle_pins.py (identity at t = 0, norm preservation,
relative-position property, complex-multiplication form)."""
import numpy as np


def llama_inv_freq(d: int = 128, base: float = 500000.0) -> np.ndarray:
    """base^(-2i/d), i < d/2, rounded to fp32 (the table the caller passes)."""
    return (base ** (-np.arange(0, d, 2, dtype=np.float64) / d)).astype(np.float32)


def rope(x: np.ndarray, pos: int, inv_freq: np.ndarray) -> np.ndarray:
    """x: [..., D] float64; returns the rotated copy (float64)."""
    x = np.asarray(x, dtype=np.float64)
    half = x.shape[-1] // 2
    theta = float(pos) * np.asarray(inv_freq, dtype=np.float64)
    c, s = np.cos(theta), np.sin(theta)
    x0, x1 = x[..., :half], x[..., half:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)
