"""Pin the CPU oracle against outputs of the reference itself (golden
fixtures from tests/golden/make_golden.py). Integer results and the C
restatement of the numba kernels must match bit for bit."""

import numpy as np
import pytest

from conftest import assert_close_rel, case_factors, golden, random_cases
from oracle import alto_oracle as orc


def test_layout_schedules_and_linearize():
    g = golden("layouts")
    i = 0
    while f"dims{i}" in g:
        dims = tuple(int(x) for x in g[f"dims{i}"])
        sched = [tuple(int(v) for v in p) for p in g[f"sched{i}"]]
        assert orc.schedule(dims) == sched
        keys = orc.encode(dims, g[f"pts{i}"])
        want = [int(s) for s in g[f"lin{i}"]]
        if keys.ndim == 1:
            got = [int(k) for k in keys]
        else:
            got = [int(k[0]) | (int(k[1]) << 64) for k in keys]
        assert got == want
        assert np.array_equal(orc.decode(dims, keys), g[f"pts{i}"])
        i += 1
    assert i >= 10


def test_worked_example():
    g = golden("worked")
    dims = tuple(g["dims"])
    keys, vals, coords = orc.from_coo(dims, g["coo_coords"], g["coo_values"])
    assert keys.tolist() == [2, 15, 20, 25, 42, 51]
    assert np.array_equal(keys, g["positions"])
    assert np.array_equal(vals, g["values"])
    bounds, lo, hi, _ = orc.segments(coords, 2)
    assert np.array_equal(lo, g["L2_lo"]) and np.array_equal(hi, g["L2_hi"])
    ones = [np.ones((d, 1)) for d in dims]
    for strategy in ("sequential", "recursive", "output"):
        assert orc.mttkrp(coords, vals, ones, 0, strategy, 2).ravel().tolist() == [1, 5, 4, 11]


@pytest.mark.parametrize("case", random_cases())
def test_encoder_partition_views(case):
    g = golden(case)
    dims = tuple(int(x) for x in g["dims"])
    cc, cv = orc.canonicalize(g["in_coords"], g["in_values"])
    assert np.array_equal(cc, g["coo_coords"]) and np.array_equal(cv, g["coo_values"])
    keys, vals, coords = orc.from_coo(dims, cc, cv)
    assert np.array_equal(keys, g["positions"])
    assert np.array_equal(vals, g["values"])
    assert np.array_equal(coords, g["coords"])
    for L in (1, 2, 4, 7):
        bounds, lo, hi, boundary = orc.segments(coords, L)
        assert np.array_equal(bounds, g[f"L{L}_bounds"])
        assert np.array_equal(lo, g[f"L{L}_lo"]) and np.array_equal(hi, g[f"L{L}_hi"])
        for n in range(len(dims)):
            assert np.array_equal(boundary[n], g[f"L{L}_boundary{n}"])
        # the argsort-free variant used at BASELINE sizes (tests/parity_full.py)
        b2, lo2, hi2, boundary2 = orc.segments_large(coords, L)
        assert np.array_equal(b2, bounds) and np.array_equal(lo2, lo) and np.array_equal(hi2, hi)
        for n in range(len(dims)):
            assert np.array_equal(boundary2[n], g[f"L{L}_boundary{n}"])
    for mode in range(len(dims)):
        for L in (2, 4, 7):
            perm, _, _, _, b = orc.mode_view(coords, vals, mode, L)
            assert np.array_equal(perm, g[f"view{L}_m{mode}_perm"])
            assert np.array_equal(b, g[f"view{L}_m{mode}_boundary"])


@pytest.mark.parametrize("case", random_cases())
def test_kernels_bitwise(case):
    g = golden(case)
    dims = tuple(int(x) for x in g["dims"])
    coords, vals = g["coords"], g["values"]
    factors = case_factors(g)
    for mode in range(len(dims)):
        assert np.array_equal(orc.mttkrp(coords, vals, factors, mode), g[f"seq_m{mode}"])
        scaled = g[f"scaled_m{mode}"]
        assert np.array_equal(orc.pi_rows(coords, factors, mode), g[f"pi_m{mode}"])
        assert np.array_equal(orc.phi(coords, vals, scaled, factors, mode), g[f"phiseq_m{mode}"])
        pre = orc.phi(coords, vals, scaled, factors, mode, krp_rows=g[f"pi_m{mode}"])
        assert np.array_equal(pre, g[f"phiseq_m{mode}"])
        for L in (2, 4, 7):
            assert np.array_equal(orc.mttkrp(coords, vals, factors, mode, "recursive", L, 2),
                                  g[f"rec{L}_m{mode}"])
            assert np.array_equal(orc.mttkrp(coords, vals, factors, mode, "output", L),
                                  g[f"out{L}_m{mode}"])
            assert np.array_equal(orc.phi(coords, vals, scaled, factors, mode, "recursive", L, threads=2),
                                  g[f"phirec{L}_m{mode}"])
            assert np.array_equal(orc.phi(coords, vals, scaled, factors, mode, "output", L),
                                  g[f"phiout{L}_m{mode}"])


def test_wide_128bit_and_duplicates():
    g = golden("wide128")
    dims = tuple(int(x) for x in g["dims"])
    cc, cv = orc.canonicalize(g["in_coords"], g["in_values"])
    keys, vals, coords = orc.from_coo(dims, cc, cv)
    assert keys.shape[1] == 2
    assert np.array_equal(keys, g["positions"]) and np.array_equal(vals, g["values"])
    factors = [np.random.default_rng(int(s)).random((d, 4)) for s, d in zip(g["factor_seeds"], dims)]
    for mode in range(4):
        out = orc.mttkrp(coords, vals, factors, mode)
        rows = g[f"seq_m{mode}_rows"]
        assert np.array_equal(out[rows], g[f"seq_m{mode}_vals"])
    d = golden("duplicates")
    cc, cv = orc.canonicalize(d["in_coords"], d["in_values"])
    assert np.array_equal(cc, d["coo_coords"]) and np.array_equal(cv, d["coo_values"])


def test_drivers_against_reference():
    g = golden("drivers")
    dims = tuple(int(x) for x in g["dims"])
    coords, vals = g["coords"], g["values"]
    for tag, strategy, L in (("seq", "sequential", 1), ("rec", "recursive", 2)):
        w, fs, fits = orc.cp_als(dims, coords, vals, 3, 6, seed=5, fit_tol=1e-14, strategy=strategy, L=L,
                                 threads=2)
        assert_close_rel(fits, g[f"als_{tag}_fit"], rel=1e-12)
        assert_close_rel(w, g[f"als_{tag}_weights"], rel=1e-12)
        for n, f in enumerate(fs):
            assert_close_rel(f, g[f"als_{tag}_factor{n}"], rel=1e-12)
    adims = tuple(int(x) for x in g["apr_dims"])
    for tag, kw in (("otf", {}), ("pre", {"pre": True}), ("rec", {"strategy": "recursive", "L": 2})):
        w, fs, kkts, inners, lls = orc.cp_apr(adims, g["apr_coords"], g["apr_values"], 2, 12, seed=2, **kw)
        assert np.array_equal(np.asarray(inners), g[f"apr_{tag}_inner"])
        assert_close_rel(lls, g[f"apr_{tag}_loglik"], rel=1e-12)
        assert_close_rel(w, g[f"apr_{tag}_weights"], rel=1e-12)
        for n, f in enumerate(fs):
            assert_close_rel(f, g[f"apr_{tag}_factor{n}"], rel=1e-12)
    _, init = orc.init_factors((4, 8, 2), 2, seed=42)
    for n, f in enumerate(init):
        assert np.array_equal(f, g[f"init42_factor{n}"])
