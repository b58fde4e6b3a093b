"""Seeded synthetic stand-ins for the BASELINE.json configs.

No public dataset is named by BASELINE; the paper's FROSTT tensors are not
available, so these generators reproduce each config's shape, nonzero count
and value/coordinate distributions (SURVEY.md §8(d) "Generator rules"):

* coordinates per mode uniform, or Zipf(alpha) truncated to ranks 1..I_n
  (P(k) ~ k^-alpha) mapped through a seeded random permutation of the mode;
* draws are made in batches and deduplicated (the GPU canonicaliser), until
  at least M unique coordinates exist; exactly M are then selected uniformly;
* values are drawn after selection; U(0,1) draws of exactly 0 are resampled.

Two backends: ``generate`` (torch on the GPU, full BASELINE sizes) and
``generate_numpy`` (host, for bounded CPU-baseline samples). They share the
distribution, not the random stream.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    nnz: int
    coord_dist: tuple  # per mode: ("uniform",) or ("zipf", alpha)
    values: str  # "uniform" | "lognormal" | "poisson1p2"
    rank: int
    description: str


CONFIGS = {
    "c1": Config("c1", (1000, 1000, 1000), 1_000_000, (("uniform",),) * 3, "uniform", 16,
                 "3-mode 1000^3, 1M uniform nnz, R=16 (BASELINE configs[0])"),
    "c2": Config("c2", (12000, 9000, 28000), 76_000_000, (("zipf", 1.2),) * 3, "uniform", 16,
                 "3-mode 12000x9000x28000, 76M Zipf(1.2) nnz, R=16, CP-ALS (BASELINE configs[1])"),
    "c3": Config("c3", (2_000_000, 2_000_000, 2_000_000, 168), 140_000_000,
                 (("zipf", 1.1),) * 3 + (("uniform",),), "lognormal", 32,
                 "4-mode 2Mx2Mx2Mx168, 140M nnz, long modes Zipf(1.1), R=32 (BASELINE configs[2])"),
    "c4": Config("c4", (50000, 50000, 5000), 50_000_000, (("zipf", 1.3),) * 3, "poisson1p2", 10,
                 "3-mode 50000x50000x5000 counts, 50M Zipf(1.3) nnz, R=10, CP-APR (BASELINE configs[3])"),
    "c5": Config("c5", (10_000_000, 10_000_000, 1_000_000, 100_000, 1000), 500_000_000,
                 (("zipf", 1.05),) * 5, "uniform", 32,
                 "5-mode hypersparse, 500M Zipf(1.05) nnz, R=32, 128-bit keys (BASELINE configs[4])"),
}


def _zipf_cdf_np(n: int, alpha: float) -> np.ndarray:
    w = np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
    c = np.cumsum(w)
    return c / c[-1]


def generate(cfg: Config, seed: int = 0, nnz: int | None = None, batch_factor: float = 2.0):
    """GPU generator -> (device coords (M, N) int64, device values (M,) f64),
    unique coordinates in random order."""
    import torch

    from . import _native as nat
    from .encoding import lexicographic_layout
    from .tensor import _canonicalize

    dev = nat.device()
    M = cfg.nnz if nnz is None else int(nnz)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    N = len(cfg.dims)
    perms, cdfs = [], []
    for n, d in enumerate(cfg.dims):
        dist = cfg.coord_dist[n]
        if dist[0] == "zipf":
            perms.append(torch.randperm(d, generator=g, device=dev))
            cdfs.append(torch.from_numpy(_zipf_cdf_np(d, dist[1])).to(dev))
        else:
            perms.append(None)
            cdfs.append(None)
    from .encoding import as_shape

    shape = as_shape(cfg.dims)
    if M * N * 8 > _LEAN_BYTES:
        coords = _unique_coords_lean(cfg, shape, M, g, dev, perms, cdfs)
        return coords, _values_torch(cfg.values, M, g, dev)
    uniq = torch.empty((0, N), dtype=torch.int64, device=dev)
    draws = max(int(M * batch_factor), 1024)
    for _ in range(64):
        cols = []
        for n, d in enumerate(cfg.dims):
            if cdfs[n] is None:
                cols.append(torch.randint(0, d, (draws,), generator=g, device=dev, dtype=torch.int64))
            else:
                u = torch.rand(draws, generator=g, device=dev, dtype=torch.float64)
                r = torch.searchsorted(cdfs[n], u, right=True).clamp_(max=d - 1)
                cols.append(perms[n][r])
        batch = torch.stack(cols, dim=1)
        del cols
        allc = torch.cat([uniq, batch], dim=0)
        del batch
        ones = torch.ones(allc.shape[0], dtype=torch.float64, device=dev)
        uniq, _v = _canonicalize(shape, allc, ones)
        del allc, ones, _v
        if uniq.shape[0] >= M:
            break
        # yield shrinks as the head saturates: grow the next batch
        draws = int(draws * 1.5)
    if uniq.shape[0] < M:
        raise RuntimeError(f"could not draw {M} unique coordinates for {cfg.name}")
    pick = torch.randperm(uniq.shape[0], generator=g, device=dev)[:M]
    coords = uniq.index_select(0, pick).contiguous()
    del uniq, pick
    values = _values_torch(cfg.values, M, g, dev)
    return coords, values


# coordinate arrays above this size (c5: 500M x 5 int64 = 20 GB) are drawn
# through the memory-lean path below; smaller configs keep the original
# stream (their seeded data is unchanged)
_LEAN_BYTES = 8 << 30


def _draw_cols(cfg, n_draws, g, dev, perms, cdfs):
    import torch

    cols = []
    for n, d in enumerate(cfg.dims):
        if cdfs[n] is None:
            cols.append(torch.randint(0, d, (n_draws,), generator=g, device=dev, dtype=torch.int64))
        else:
            u = torch.rand(n_draws, generator=g, device=dev, dtype=torch.float64)
            r = torch.searchsorted(cdfs[n], u, right=True).clamp_(max=d - 1)
            cols.append(perms[n][r])
    return torch.stack(cols, dim=1)


def _unique_coords_lean(cfg, shape, M, g, dev, perms, cdfs):
    """Unique coordinates kept as lexicographic keys (16 B instead of 8N B
    per entry): draw in bounded batches, encode, sort + drop duplicates on
    the device, decode only the M selected at the end."""
    import torch

    from .encoding import lexicographic_layout
    from .tensor import device_decode, device_encode, sort_pairs

    lay = lexicographic_layout(shape)
    uniq = None
    chunk = 64 << 20  # coordinates drawn per encode step
    target = int(M * 1.05)
    for _ in range(64):
        have = 0 if uniq is None else uniq.shape[0]
        need = max(target - have, 1 << 20)
        parts = [] if uniq is None else [uniq]
        left = int(need * 1.3)
        while left > 0:
            n = min(left, chunk)
            parts.append(device_encode(lay, _draw_cols(cfg, n, g, dev, perms, cdfs)))
            left -= n
        keys = torch.cat(parts, dim=0)
        del parts, uniq
        dummy = torch.zeros(keys.shape[0], dtype=torch.float64, device=dev)
        sort_pairs(lay, keys, dummy)
        del dummy
        if keys.ndim == 1:
            keep = torch.ones(keys.shape[0], dtype=torch.bool, device=dev)
            keep[1:] = keys[1:] != keys[:-1]
        else:
            keep = torch.ones(keys.shape[0], dtype=torch.bool, device=dev)
            keep[1:] = (keys[1:] != keys[:-1]).any(dim=1)
        uniq = keys[keep]
        del keys, keep
        if uniq.shape[0] >= M:
            break
    if uniq.shape[0] < M:
        raise RuntimeError(f"could not draw {M} unique coordinates for {cfg.name}")
    pick = torch.randperm(uniq.shape[0], generator=g, device=dev)[:M]
    sel = uniq.index_select(0, pick)
    del uniq, pick
    return device_decode(lay, sel)


def _values_torch(kind: str, M: int, g, dev):
    import torch

    if kind == "uniform":
        v = torch.rand(M, generator=g, device=dev, dtype=torch.float64)
        while True:
            z = v == 0.0
            if not bool(z.any()):
                break
            v[z] = torch.rand(int(z.sum()), generator=g, device=dev, dtype=torch.float64)
        return v
    if kind == "lognormal":
        return torch.exp(torch.randn(M, generator=g, device=dev, dtype=torch.float64))
    if kind == "poisson1p2":
        lam = torch.full((M,), 2.0, device=dev, dtype=torch.float64)
        return 1.0 + torch.poisson(lam, generator=g)
    raise ValueError(kind)


def generate_numpy(cfg: Config, nnz: int, seed: int = 0):
    """Host generator for bounded samples: (coords (M, N) int64, values)."""
    rng = np.random.default_rng(seed)
    N = len(cfg.dims)
    maps = []
    for n, d in enumerate(cfg.dims):
        dist = cfg.coord_dist[n]
        maps.append((rng.permutation(d), _zipf_cdf_np(d, dist[1])) if dist[0] == "zipf" else None)
    radix = [int(d) for d in cfg.dims]
    flat_ok = math.prod(radix) < 2**63
    seen = None
    draws = max(2 * nnz, 1024)
    for _ in range(64):
        cols = []
        for n, d in enumerate(cfg.dims):
            if maps[n] is None:
                cols.append(rng.integers(0, d, draws))
            else:
                perm, cdf = maps[n]
                r = np.minimum(np.searchsorted(cdf, rng.random(draws), side="right"), d - 1)
                cols.append(perm[r])
        c = np.stack(cols, axis=1).astype(np.int64)
        c = c if seen is None else np.concatenate([seen, c])
        if flat_ok:
            flat = np.ravel_multi_index(tuple(c.T), cfg.dims)
            _, idx = np.unique(flat, return_index=True)
            seen = c[np.sort(idx)]
        else:
            seen = np.unique(c, axis=0)
        if seen.shape[0] >= nnz:
            break
        draws = int(draws * 1.5)
    pick = rng.permutation(seen.shape[0])[:nnz]
    coords = seen[pick]
    if cfg.values == "uniform":
        v = rng.random(nnz)
        while (v == 0.0).any():
            v[v == 0.0] = rng.random(int((v == 0.0).sum()))
    elif cfg.values == "lognormal":
        v = np.exp(rng.standard_normal(nnz))
    else:
        v = 1.0 + rng.poisson(2.0, nnz).astype(np.float64)
    return coords, v


def algorithmic_bytes(cfg_or_dims, nnz: int, rank: int, key_bytes: int, kind: str = "mttkrp",
                      mode: int = 0) -> int:
    """Compulsory traffic per launch:
    MTTKRP  M (W + 8) + 8 R sum_m I_m
    Phi OTF M (W + 8) + 8 R (sum_{m != n} I_m + 2 I_n)
    loglik  M (W + 8) + 8 R sum_m I_m
    Phi PRE M (W + 8) + 8 M R + 16 I_n R   (kind "phi_pre")"""
    dims = cfg_or_dims.dims if hasattr(cfg_or_dims, "dims") else tuple(cfg_or_dims)
    stream = nnz * (key_bytes + 8)
    if kind == "phi_pre":
        return stream + 8 * nnz * rank + 16 * dims[mode] * rank
    if kind == "phi":
        return stream + 8 * rank * (sum(dims) - dims[mode] + 2 * dims[mode])
    return stream + 8 * rank * sum(dims)
