"""The hand-written stable LSD radix sort (csrc/radix_sort.cu) against numpy's
stable argsort / lexsort: exact permutation (stability included) for 64- and
128-bit keys, every digit count, tile-edge sizes, heavy duplication."""

import numpy as np
import pytest
import torch

from paper_2403_06348_b200.encoding import build_layout
from paper_2403_06348_b200.tensor import sort_pairs

pytestmark = pytest.mark.gpu

# dims -> total_bits: (2,) 1; (128,) 7; (256,) 8; (2^21, 2^22) 43; (2^32, 2^32) 64;
# 2M^3 x 168 (c3) 71; c5 95; (2^64-ish) 128 via four 2^32 modes
SHAPES64 = [(2,), (128,), (256,), (2**21, 2**22), (2**32, 2**32)]
SHAPES128 = [(2_000_000, 2_000_000, 2_000_000, 168), (10_000_000, 10_000_000, 1_000_000, 100_000, 1000),
             (2**32, 2**32, 2**32, 2**32)]
SIZES = [2, 100, 4095, 4096, 4097, 100_003, 1_000_000]


def _keys(rng, bits, M, dup):
    if dup:  # few distinct values -> long equal runs (stability)
        base = rng.integers(0, 2**min(bits, 62), size=max(M // 50, 1), dtype=np.uint64)
        return base[rng.integers(0, base.size, size=M)]
    if bits == 64:
        return rng.integers(0, 2**63, size=M, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=M, dtype=np.uint64)
    return rng.integers(0, 2**bits, size=M, dtype=np.uint64)


@pytest.mark.parametrize("dims", SHAPES64)
@pytest.mark.parametrize("M", SIZES)
def test_sort64_matches_stable_argsort(dims, M):
    lay = build_layout(dims)
    assert lay.word_bits == 64
    rng = np.random.default_rng(M + lay.total_bits)
    for dup in (False, True):
        k = _keys(rng, lay.total_bits, M, dup)
        order = np.argsort(k, kind="stable")
        dk = torch.from_numpy(k.view(np.int64).copy()).cuda()
        dv = torch.arange(M, dtype=torch.float64, device="cuda")
        sort_pairs(lay, dk, dv)
        assert np.array_equal(dk.cpu().numpy().view(np.uint64), k[order])
        assert np.array_equal(dv.cpu().numpy().astype(np.int64), order)


@pytest.mark.parametrize("dims", SHAPES128)
@pytest.mark.parametrize("M", [2, 4097, 300_001])
def test_sort128_matches_lexsort(dims, M):
    lay = build_layout(dims)
    assert lay.word_bits == 128
    rng = np.random.default_rng(M + lay.total_bits)
    hi_bits = lay.total_bits - 64
    for dup in (False, True):
        lo = _keys(rng, 64, M, dup)
        hi = _keys(rng, hi_bits, M, dup)
        if dup:  # equal (lo, hi) pairs
            lo[1::3] = lo[0:-1:3][: lo[1::3].size]
            hi[1::3] = hi[0:-1:3][: hi[1::3].size]
        order = np.lexsort((lo, hi))  # stable, hi major
        pairs = np.stack([lo, hi], axis=1)
        dk = torch.from_numpy(pairs.view(np.int64).copy()).cuda()
        dv = torch.arange(M, dtype=torch.float64, device="cuda")
        sort_pairs(lay, dk, dv)
        assert np.array_equal(dk.cpu().numpy().view(np.uint64), pairs[order])
        assert np.array_equal(dv.cpu().numpy().astype(np.int64), order)
