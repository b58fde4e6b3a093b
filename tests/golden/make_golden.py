"""Generate golden fixtures by running the REFERENCE implementation.

Runs only in the build container (needs /root/reference); the outputs are
committed as tests/golden/*.npz and travel to the GPU box. Usage:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Inputs are seeded numpy draws made here; every output array is what the
reference package (pkg/src/alto) computes for them.
"""

from __future__ import annotations

import io
import math
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

import alto  # noqa: E402  (the reference package)
from alto.cpd import CpAlsConfig, CpAprConfig, KruskalModel, cp_als, cp_apr_mu  # noqa: E402
from alto.cpd.apr import phi_kernel, precompute_krp_rows  # noqa: E402
from alto.encoding import build_layout, linearize  # noqa: E402
from alto.kernels import mttkrp_output_oriented, mttkrp_recursive, mttkrp_sequential  # noqa: E402
from alto.partition import make_mode_ordered_view, make_segments  # noqa: E402

OUT = Path(__file__).resolve().parent

EXAMPLE_TNS = "1 4 1 1\n2 1 1 2\n2 7 2 3\n3 3 2 4\n4 2 2 5\n4 5 1 6\n"


def random_sparse(rng, dims, nnz, kind="positive"):
    total = math.prod(int(k) for k in dims)
    nnz = min(nnz, total)
    if total <= 2**24:
        flat = rng.choice(total, size=nnz, replace=False)
        coords = np.stack(np.unravel_index(flat, dims), axis=1)
    else:
        coords = np.stack([rng.integers(0, d, size=nnz) for d in dims], axis=1)
    if kind == "counts":
        values = rng.integers(1, 10, size=nnz).astype(np.float64)
    else:
        values = rng.random(nnz) + 0.05
    return coords.astype(np.int64), values


def segs_record(d, prefix, t, L):
    s = make_segments(t, L)
    d[f"{prefix}_bounds"] = s.bounds()
    d[f"{prefix}_lo"] = np.asarray([[iv[0] for iv in seg.intervals] for seg in s.segments])
    d[f"{prefix}_hi"] = np.asarray([[iv[1] for iv in seg.intervals] for seg in s.segments])
    d[f"{prefix}_pos_first"] = np.asarray([seg.pos_first for seg in s.segments], dtype=object).astype(str)
    d[f"{prefix}_pos_last"] = np.asarray([seg.pos_last for seg in s.segments], dtype=object).astype(str)
    for n in range(t.ndim):
        d[f"{prefix}_boundary{n}"] = np.asarray(s.boundary_rows[n], dtype=np.int64)


def worked():
    coo = alto.parse_frostt(io.StringIO(EXAMPLE_TNS), dims=(4, 8, 2))
    t = alto.AltoTensor.from_coo(coo)
    d = {
        "dims": np.asarray((4, 8, 2)),
        "coo_coords": coo.coords,
        "coo_values": coo.values,
        "positions": t.positions,
        "values": t.values,
        "coords": t.coords,
        "schedule": np.asarray(t.layout.schedule),
    }
    segs_record(d, "L2", t, 2)
    ones = [np.ones((k, 1)) for k in (4, 8, 2)]
    d["ones_mode0"] = mttkrp_sequential(t, ones, 0)
    v = make_mode_ordered_view(t, 0, 2)
    d["view0_coords"] = v.coords
    d["view0_perm"] = v.perm
    np.savez_compressed(OUT / "worked.npz", **d)


def random_cases():
    rng = np.random.default_rng(20240306)
    cases = []
    for i in range(14):
        ndim = 3 + i % 3
        dims = tuple(int(x) for x in rng.integers(2, 21, size=ndim))
        nnz = int(rng.integers(10, 501))
        coords, values = random_sparse(rng, dims, nnz, "counts" if i % 4 == 3 else "positive")
        rank = [1, 2, 5, 8, 16, 3, 10][i % 7]
        cases.append((dims, coords, values, rank))
    # a larger one so segments hold many rows
    dims = (60, 45, 70)
    coords, values = random_sparse(rng, dims, 2500)
    cases.append((dims, coords, values, 16))
    for i, (dims, coords, values, rank) in enumerate(cases):
        coo = alto.CooTensor(dims, coords, values)
        t = alto.AltoTensor.from_coo(coo)
        d = {
            "dims": np.asarray(dims),
            "in_coords": coords,
            "in_values": values,
            "coo_coords": coo.coords,
            "coo_values": coo.values,
            "positions": t.positions,
            "values": t.values,
            "coords": t.coords,
            "rank": np.asarray(rank),
        }
        frng = np.random.default_rng(1000 + i)
        factors = [frng.random((k, rank)) + 0.05 for k in dims]
        for n, f in enumerate(factors):
            d[f"factor{n}"] = f
        for L in (1, 2, 4, 7):
            segs_record(d, f"L{L}", t, L)
        for mode in range(len(dims)):
            d[f"seq_m{mode}"] = mttkrp_sequential(t, factors, mode)
            scaled = frng.random((dims[mode], rank)) + 0.01
            d[f"scaled_m{mode}"] = scaled
            d[f"pi_m{mode}"] = precompute_krp_rows(t, factors, mode)
            d[f"phiseq_m{mode}"] = phi_kernel(t, scaled, factors, mode, strategy="sequential")
            for L in (2, 4, 7):
                segs = make_segments(t, L)
                d[f"rec{L}_m{mode}"] = mttkrp_recursive(t, segs, factors, mode, workers=2)
                view = make_mode_ordered_view(t, mode, L)
                d[f"out{L}_m{mode}"] = mttkrp_output_oriented(t, view, factors, mode, workers=2)
                d[f"view{L}_m{mode}_boundary"] = view.boundary_rows
                d[f"view{L}_m{mode}_perm"] = view.perm
                d[f"phirec{L}_m{mode}"] = phi_kernel(t, scaled, factors, mode, workers=2,
                                                     num_segments=L, strategy="recursive")
                d[f"phiout{L}_m{mode}"] = phi_kernel(t, scaled, factors, mode, workers=2,
                                                     num_segments=L, strategy="output")
        np.savez_compressed(OUT / f"random{i:02d}.npz", **d)


def wide_and_duplicates():
    rng = np.random.default_rng(7)
    dims = (2**18, 2**17, 2**17, 2**17)
    coords, values = random_sparse(rng, dims, 300)
    coo = alto.CooTensor(dims, coords, values)
    t = alto.AltoTensor.from_coo(coo)
    factors = [np.random.default_rng(70 + n).random((k, 4)) for n, k in enumerate(dims)]
    d = {"dims": np.asarray(dims), "in_coords": coords, "in_values": values,
         "positions": t.positions, "values": t.values, "coords": t.coords,
         "factor_seeds": np.arange(70, 74)}
    for mode in range(4):
        out = mttkrp_sequential(t, factors, mode)
        rows = np.unique(t.coords[:, mode])
        d[f"seq_m{mode}_rows"] = rows
        d[f"seq_m{mode}_vals"] = out[rows]
        assert np.count_nonzero(np.delete(out, rows, axis=0)) == 0
    segs_record(d, "L3", t, 3)
    np.savez_compressed(OUT / "wide128.npz", **d)

    # duplicates, cancellation to exact zero, unsorted input
    dims = (5, 4, 6)
    base = rng.integers(0, 4, size=(40, 3))
    coords = np.concatenate([base, base[:15], base[5:10]])
    values = np.concatenate([rng.standard_normal(40), rng.standard_normal(15), rng.standard_normal(5)])
    values[40:43] = -values[0:3]  # 3 duplicates that may cancel
    coo = alto.CooTensor(dims, coords, values)
    np.savez_compressed(OUT / "duplicates.npz", dims=np.asarray(dims), in_coords=coords,
                        in_values=values, coo_coords=coo.coords, coo_values=coo.values)


def layouts():
    shapes = [(4, 8, 2), (1000, 1000, 1000), (12000, 9000, 28000), (2_000_000, 2_000_000, 2_000_000, 168),
              (50000, 50000, 5000), (10_000_000, 10_000_000, 1_000_000, 100_000, 1000), (1, 1, 1),
              (4, 4), (3, 5, 7, 2), (2**20,) * 6]
    d = {}
    rng = np.random.default_rng(11)
    for i, s in enumerate(shapes):
        lay = build_layout(s)
        d[f"dims{i}"] = np.asarray(s)
        d[f"sched{i}"] = np.asarray(lay.schedule, dtype=np.int64).reshape(-1, 2)
        pts = np.stack([rng.integers(0, k, size=20) for k in s], axis=1)
        d[f"pts{i}"] = pts
        d[f"lin{i}"] = np.asarray([str(linearize(lay, p)) for p in pts])
    np.savez_compressed(OUT / "layouts.npz", **d)


def drivers():
    rng = np.random.default_rng(17)
    dims = (8, 6, 7)
    coords, values = random_sparse(rng, dims, 120)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, values))
    d = {"dims": np.asarray(dims), "coords": t.coords, "values": t.values, "positions": t.positions}
    for tag, cfg in (("seq", CpAlsConfig(rank=3, max_iters=6, fit_tol=1e-14, seed=5)),
                     ("rec", CpAlsConfig(rank=3, max_iters=6, fit_tol=1e-14, seed=5, workers=2,
                                         num_segments=2, strategy="recursive"))):
        r = cp_als(t, cfg)
        d[f"als_{tag}_fit"] = np.asarray(r.fit_trace)
        d[f"als_{tag}_obj"] = np.asarray(r.objective_trace)
        d[f"als_{tag}_weights"] = r.model.weights
        for n, f in enumerate(r.model.factors):
            d[f"als_{tag}_factor{n}"] = f
    # CP-APR on a count tensor drawn from a stochastic model
    crng = np.random.default_rng(9)
    cdims = (5, 4, 3)
    fs = [crng.dirichlet(np.ones(k), size=2).T for k in cdims]
    w = 25.0 * (0.5 + crng.random(2))
    dense = crng.poisson(KruskalModel(w, fs).to_dense()).astype(float)
    ct = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(dense))
    d["apr_dims"] = np.asarray(cdims)
    d["apr_coords"] = ct.coords
    d["apr_values"] = ct.values
    for tag, cfg in (("otf", CpAprConfig(rank=2, seed=2, max_outer=12)),
                     ("pre", CpAprConfig(rank=2, seed=2, max_outer=12, memory_mode="pre")),
                     ("rec", CpAprConfig(rank=2, seed=2, max_outer=12, workers=2, num_segments=2,
                                         strategy="recursive"))):
        r = cp_apr_mu(ct, cfg)
        d[f"apr_{tag}_kkt"] = np.asarray(r.kkt_trace)
        d[f"apr_{tag}_inner"] = np.asarray(r.inner_iters)
        d[f"apr_{tag}_loglik"] = np.asarray(r.loglik_trace)
        d[f"apr_{tag}_weights"] = r.model.weights
        for n, f in enumerate(r.model.factors):
            d[f"apr_{tag}_factor{n}"] = f
    init = alto.init_factors((4, 8, 2), 2, seed=42)
    for n, f in enumerate(init.factors):
        d[f"init42_factor{n}"] = f
    np.savez_compressed(OUT / "drivers.npz", **d)


if __name__ == "__main__":
    worked()
    random_cases()
    wide_and_duplicates()
    layouts()
    drivers()
    print("golden fixtures written to", OUT)
