"""Dense R x R algebra for the drivers (pkg/src/alto/cpd/linalg.py:8-52).

Host versions keep the reference API; the ``*_dev`` variants operate on the
device-resident factor matrices (cuBLAS/cuSOLVER through torch -- plain
library dense algebra, not the hot path). The R x R factorisation itself is
done on the host with scipy exactly like the reference, so the
Cholesky-vs-eigh decision is identical.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

PINV_RTOL = 1e-12


def gram(factor) -> np.ndarray:
    factor = np.asarray(factor, dtype=np.float64)
    return factor.T @ factor


def hadamard_chain(grams, skip: int | None = None) -> np.ndarray:
    out = None
    for n, g in enumerate(grams):
        if n == skip:
            continue
        out = g.copy() if out is None else out * g
    if out is None:
        rank = grams[skip].shape[0]
        return np.ones((rank, rank), dtype=np.float64)
    return out


def _factorize(v: np.ndarray):
    """('chol', c) or ('pinv', P) for the symmetric PSD matrix v."""
    try:
        c, low = scipy.linalg.cho_factor(v)
        return "chol", (c, low)
    except scipy.linalg.LinAlgError:
        pass
    w, u = scipy.linalg.eigh(v)
    cutoff = PINV_RTOL * max(w.max(), 0.0)
    inv = np.zeros_like(w)
    keep = w > cutoff
    inv[keep] = 1.0 / w[keep]
    return "pinv", (u * inv) @ u.T


def solve_pseudo(mat, v) -> np.ndarray:
    mat = np.asarray(mat, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if not (np.isfinite(mat).all() and np.isfinite(v).all()):
        raise ValueError("non-finite input to the normal-equation solve")
    kind, f = _factorize(v)
    if kind == "chol":
        return scipy.linalg.cho_solve(f, mat.T).T
    return mat @ f


def gram_dev(a) -> np.ndarray:
    """A^T A of a device (rows, R) matrix, returned on the host."""
    return (a.T @ a).cpu().numpy()


def solve_pseudo_dev(mat, v: np.ndarray, check_finite: bool = True):
    """mat @ pinv(v) for a device (rows, R) mat; v on host (R x R).
    ``check_finite=False`` skips the device-side scan of ``mat`` (a host
    sync); the caller must then detect non-finite results itself."""
    import torch

    if (check_finite and not bool(torch.isfinite(mat).all())) or not np.isfinite(v).all():
        raise ValueError("non-finite input to the normal-equation solve")
    kind, f = _factorize(np.asarray(v, dtype=np.float64))

    def upload(x):
        # pinned + non_blocking: the host does not wait for the queued kernels
        return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().to(mat.device, non_blocking=True)

    if kind == "chol":
        c, low = f
        tri = np.tril(c) if low else np.triu(c).T  # lower factor L with v = L L^T
        return torch.cholesky_solve(mat.T.contiguous(), upload(tri), upper=False).T
    return mat @ upload(f)
