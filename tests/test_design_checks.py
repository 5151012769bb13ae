"""Host-side checks of the kernel's index design (no GPU): the token
permutation is a bijection, every MMA k-slot maps to one head dim, and every
fragment read from the 128B-swizzled tiles is bank-conflict free."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import check_banks as cb  # noqa: E402


def test_token_permutation_is_bijection():
    rows = [cb.tok_pi(r) for r in range(8)] + [8 + cb.tok_pi(r) for r in range(8)]
    assert sorted(rows) == list(range(16))


def test_k_dims_cover_each_mma_once():
    # MMA jj uses chunk i = jj // 2 (q + 4i) and words 2*(jj&1), +1 -> 4 dims per thread q
    for jj in range(8):
        dims = []
        for q in range(4):
            c = q + 4 * (jj >> 1)
            w = 2 * (jj & 1)
            dims += [8 * c + 2 * w, 8 * c + 2 * w + 1, 8 * c + 2 * w + 2, 8 * c + 2 * w + 3]
        assert len(set(dims)) == 16
    allc = sorted(q + 4 * i for q in range(4) for i in range(4))
    assert allc == list(range(16))


def test_v_rows_cover_all_dims():
    dims = sorted(d for r in range(8) for i in range(8) for d in (8 * r + i, 64 + 8 * r + i))
    assert dims == list(range(128))


def test_fragment_reads_conflict_free():
    assert cb.main() == (1, 1)
