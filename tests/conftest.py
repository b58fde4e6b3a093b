import math
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"

EXAMPLE_DIMS = (4, 8, 2)
EXAMPLE_COORDS = [[0, 3, 0], [1, 0, 0], [1, 6, 1], [2, 2, 1], [3, 1, 1], [3, 4, 0]]
EXAMPLE_VALUES = [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def random_cases():
    return sorted(p.stem for p in GOLDEN.glob("random*.npz"))


def case_factors(g):
    n = len(g["dims"])
    return [g[f"factor{i}"] for i in range(n)]


def assert_close_rel(got, want, rel=1e-12, scale=None):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if scale is None:
        scale = max(float(np.abs(want).max(initial=0.0)), 1e-300)
    err = float(np.abs(got - want).max(initial=0.0))
    assert err <= rel * scale, f"max abs err {err} > {rel} * {scale}"


def assert_monotone(seq, direction="nonincreasing", rel=1e-9, floor=1e-30):
    seq = np.asarray(seq, dtype=np.float64)
    slack = rel * np.maximum(np.abs(seq[:-1]), floor)
    diff = np.diff(seq)
    bad = diff > slack if direction == "nonincreasing" else diff < -slack
    assert not bad.any(), f"sequence not {direction}: {seq.tolist()}"


def random_sparse(rng, dims, nnz, kind="normal"):
    """Distinct coordinates, nonzero values (same recipe as the reference
    test helper, pkg/tests/conftest.py:31-48)."""
    total = math.prod(dims)
    nnz = min(nnz, total)
    if total <= 2**24:
        flat = rng.choice(total, size=nnz, replace=False)
        coords = np.stack(np.unravel_index(flat, dims), axis=1)
    else:
        coords = np.stack([rng.integers(0, d, size=nnz) for d in dims], axis=1)
    if kind == "counts":
        values = rng.integers(1, 10, size=nnz).astype(np.float64)
    elif kind == "positive":
        values = rng.random(nnz) + 0.05
    else:
        values = rng.standard_normal(nnz)
        values[values == 0.0] = 1.0
    return coords.astype(np.int64), values


def dense_mttkrp_oracle(dense, factors, mode):
    """Matricised dense tensor times the materialised Khatri-Rao product."""
    unfolded = np.moveaxis(dense, mode, 0).reshape(dense.shape[mode], -1, order="F")
    rest = [f for m, f in enumerate(factors) if m != mode]
    cols = []
    for r in range(rest[0].shape[1]):
        col = np.ones(1)
        for f in rest:
            col = np.kron(f[:, r], col)
        cols.append(col)
    return unfolded @ np.stack(cols, axis=1)
