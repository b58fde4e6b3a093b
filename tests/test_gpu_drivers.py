"""CP-ALS and CP-APR drivers on the B200 vs the reference's own traces
(golden) -- factors, weights, fit / log-likelihood within 1e-9, CP-APR
inner-iteration counts exactly (pkg/tests/test_cpd_als.py, test_cpd_apr.py)."""

import warnings

import numpy as np
import pytest

import paper_2403_06348_b200 as alto
from conftest import assert_close_rel, assert_monotone, golden, random_sparse

pytestmark = pytest.mark.gpu


def _drivers():
    g = golden("drivers")
    dims = tuple(int(x) for x in g["dims"])
    t = alto.AltoTensor(alto.build_layout(dims), g["positions"], g["values"])
    return g, dims, t


@pytest.mark.parametrize("exact", [True, False])
def test_cp_als_matches_reference(exact):
    g, dims, t = _drivers()
    for tag, cfg in (("seq", alto.CpAlsConfig(rank=3, max_iters=6, fit_tol=1e-14, seed=5)),
                     ("rec", alto.CpAlsConfig(rank=3, max_iters=6, fit_tol=1e-14, seed=5, workers=2,
                                              num_segments=2, strategy="recursive"))):
        r = alto.cp_als(t, cfg, exact=exact)
        assert_close_rel(r.fit_trace, g[f"als_{tag}_fit"], rel=1e-9)
        assert_close_rel(r.objective_trace, g[f"als_{tag}_obj"], rel=1e-9)
        assert_close_rel(r.model.weights, g[f"als_{tag}_weights"], rel=1e-9)
        for n, f in enumerate(r.model.factors):
            assert_close_rel(f, g[f"als_{tag}_factor{n}"], rel=1e-9)


@pytest.mark.parametrize("exact", [True, False])
def test_cp_apr_matches_reference(exact):
    g = golden("drivers")
    dims = tuple(int(x) for x in g["apr_dims"])
    coords, values = g["apr_coords"], g["apr_values"]
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, values))
    for tag, cfg in (("otf", alto.CpAprConfig(rank=2, seed=2, max_outer=12)),
                     ("pre", alto.CpAprConfig(rank=2, seed=2, max_outer=12, memory_mode="pre")),
                     ("rec", alto.CpAprConfig(rank=2, seed=2, max_outer=12, workers=2, num_segments=2,
                                              strategy="recursive"))):
        r = alto.cp_apr_mu(t, cfg, exact=exact)
        assert np.array_equal(np.asarray(r.inner_iters), g[f"apr_{tag}_inner"]), tag
        assert_close_rel(r.loglik_trace, g[f"apr_{tag}_loglik"], rel=1e-9)
        assert_close_rel(np.asarray(r.kkt_trace), g[f"apr_{tag}_kkt"], rel=1e-6)
        assert_close_rel(r.model.weights, g[f"apr_{tag}_weights"], rel=1e-9)
        for n, f in enumerate(r.model.factors):
            assert_close_rel(f, g[f"apr_{tag}_factor{n}"], rel=1e-9)


def test_rank_one_recovery_and_zero_iterations():
    rng = np.random.default_rng(12)
    for seed in range(3):
        true = alto.KruskalModel(np.array([1.5]), [rng.random((4, 1)) + 0.1, rng.random((3, 1)) + 0.1,
                                                   rng.random((5, 1)) + 0.1])
        t = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(true.to_dense()))
        r = alto.cp_als(t, alto.CpAlsConfig(rank=1, max_iters=25, fit_tol=1e-14, seed=seed))
        assert r.fit >= 0.9999
    coords, vals = random_sparse(rng, (4, 3, 5), 30)
    t = alto.AltoTensor.from_coo(alto.CooTensor((4, 3, 5), coords, vals))
    r = alto.cp_als(t, alto.CpAlsConfig(rank=2, max_iters=0, seed=9))
    want = alto.init_factors(t.shape, 2, seed=9).normalized(ord=2)
    for a, b in zip(r.model.factors, want.factors):
        assert np.array_equal(a, b)
    assert r.n_iters == 0 and len(r.fit_trace) == 1


def test_fit_equals_direct_and_monotone():
    rng = np.random.default_rng(14)
    coords, vals = random_sparse(rng, (4, 3, 5), 40)
    coo = alto.CooTensor((4, 3, 5), coords, vals)
    t = alto.AltoTensor.from_coo(coo)
    r = alto.cp_als(t, alto.CpAlsConfig(rank=3, max_iters=4, fit_tol=1e-14, seed=0))
    dense = coo.to_dense()
    direct = 1.0 - np.linalg.norm(dense - r.model.to_dense()) / np.linalg.norm(dense)
    assert r.fit == pytest.approx(direct, abs=1e-9)
    r = alto.cp_als(t, alto.CpAlsConfig(rank=4, max_iters=25, fit_tol=1e-14, seed=3))
    assert_monotone(r.objective_trace, "nonincreasing", rel=1e-9)


def test_apr_driver_contract():
    model = alto.KruskalModel(np.array([8.0]), [np.full((2, 1), 0.5)] * 3)
    t = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(model.to_dense()))
    res = alto.cp_apr_mu(t, alto.CpAprConfig(rank=1, seed=0), init=model)
    assert res.converged and res.n_outer == 1 and res.inner_iters == [[1, 1, 1]]
    neg = alto.AltoTensor.from_coo(alto.CooTensor((2, 2), [[0, 0], [1, 1]], [1.0, -2.0]))
    with pytest.raises(ValueError, match="negative"):
        alto.cp_apr_mu(neg, alto.CpAprConfig(rank=1))
    frac = alto.AltoTensor.from_coo(alto.CooTensor((2, 2), [[0, 0], [1, 1]], [1.5, 2.0]))
    with pytest.warns(UserWarning, match="counts"):
        alto.cp_apr_mu(frac, alto.CpAprConfig(rank=1, max_outer=2))


def test_apr_inner_loglik_monotone_and_kkt():
    rng = np.random.default_rng(8)
    dims = (5, 4, 3)
    fs = [rng.dirichlet(np.ones(d), size=2).T for d in dims]
    dense = rng.poisson(alto.KruskalModel(25.0 * (0.5 + rng.random(2)), fs).to_dense()).astype(float)
    t = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(dense))
    res = alto.cp_apr_mu(t, alto.CpAprConfig(rank=2, seed=1, track_inner_loglik=True))
    assert res.converged and res.final_kkt < 1e-4
    for sweep in res.inner_loglik:
        for inner in sweep:
            assert_monotone(inner, "nondecreasing", rel=1e-9)
    assert res.loglik_trace[-1] == pytest.approx(alto.poisson_loglik(t, res.model), rel=1e-12)
    assert (res.model.weights >= 0).all() and all((f >= 0).all() for f in res.model.factors)


def test_pre_and_otf_models_bitwise_equal(monkeypatch):
    # the gathering OTF kernel (the streamed-Pi inner iterations sum the
    # dot products in another order: tested to 1e-9 below)
    monkeypatch.setenv("ALTO_B200_PSTREAM", "0")
    rng = np.random.default_rng(11)
    dims = (5, 4, 3)
    fs = [rng.dirichlet(np.ones(d), size=2).T for d in dims]
    dense = rng.poisson(alto.KruskalModel(25.0 * (0.5 + rng.random(2)), fs).to_dense()).astype(float)
    t = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(dense))
    for exact in (True, False):
        a = alto.cp_apr_mu(t, alto.CpAprConfig(rank=2, seed=5, max_outer=3), exact=exact)
        b = alto.cp_apr_mu(t, alto.CpAprConfig(rank=2, seed=5, max_outer=3, memory_mode="pre"), exact=exact)
        assert b.memory_mode == "pre" and a.memory_mode == "otf"
        for fa, fb in zip(a.model.factors, b.model.factors):
            assert np.array_equal(fa, fb)


def test_device_driven_inner_loop_equals_host_loop(monkeypatch):
    """The device-decided inner loop (one host sync per mode) runs the same
    kernels in the same order as the host-decided one: results are bitwise
    identical, including the inner iteration counts and early breaks."""
    g = golden("drivers")
    dims = tuple(int(x) for x in g["apr_dims"])
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, g["apr_coords"], g["apr_values"]))
    cfg = alto.CpAprConfig(rank=2, seed=2, max_outer=12)
    monkeypatch.setenv("ALTO_B200_KERNEL", "dview")
    monkeypatch.setenv("ALTO_B200_PSTREAM", "0")
    dev = alto.cp_apr_mu(t, cfg)
    monkeypatch.setenv("ALTO_B200_HOST_INNER", "1")
    host = alto.cp_apr_mu(t, cfg)
    assert dev.inner_iters == host.inner_iters
    assert any(min(row) < cfg.max_inner for row in dev.inner_iters)  # breaks were exercised
    assert np.array_equal(np.asarray(dev.kkt_trace), np.asarray(host.kkt_trace))
    assert dev.loglik_trace == host.loglik_trace
    for a, b in zip(dev.model.factors, host.model.factors):
        assert np.array_equal(a, b)
    assert np.array_equal(dev.model.weights, host.model.weights)
    # exact-model one-iteration convergence through the device loop
    model = alto.KruskalModel(np.array([8.0]), [np.full((2, 1), 0.5)] * 3)
    t1 = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(model.to_dense()))
    monkeypatch.delenv("ALTO_B200_HOST_INNER")
    res = alto.cp_apr_mu(t1, alto.CpAprConfig(rank=1, seed=0), init=model)
    assert res.converged and res.n_outer == 1 and res.inner_iters == [[1, 1, 1]]


@pytest.mark.parametrize("graph", ["1", "0"])
def test_streamed_pi_inner_loop_matches_gathering_loop(monkeypatch, graph):
    """Inner iterations 2.. of every mode stream the Khatri-Rao rows stored by
    the first (csrc/pstream.cu): same inner iteration counts, KKT values,
    log-likelihoods and factors as the all-gathering device loop (1e-9),
    through the CUDA-graph outer iteration and the eager device loop, on
    the reference's golden CP-APR case and a larger skewed count tensor."""
    monkeypatch.setenv("ALTO_B200_KERNEL", "dview")
    monkeypatch.setenv("ALTO_B200_NO_GRAPH", "0" if graph == "1" else "1")
    g = golden("drivers")
    dims = tuple(int(x) for x in g["apr_dims"])
    cases = [(alto.AltoTensor.from_coo(alto.CooTensor(dims, g["apr_coords"], g["apr_values"])),
              alto.CpAprConfig(rank=2, seed=2, max_outer=12))]
    rng = np.random.default_rng(21)
    big = (300, 200, 90)
    zipf = [np.minimum(rng.zipf(1.4, 120_000) - 1, d - 1) for d in big]
    coords = np.unique(np.stack(zipf, axis=1), axis=0)
    vals = 1.0 + rng.poisson(2.0, len(coords)).astype(np.float64)
    cases.append((alto.AltoTensor.from_coo(alto.CooTensor(big, coords, vals)),
                  alto.CpAprConfig(rank=10, seed=3, max_outer=4)))
    for t, cfg in cases:
        monkeypatch.setenv("ALTO_B200_PSTREAM", "0")
        ref = alto.cp_apr_mu(t, cfg)
        monkeypatch.setenv("ALTO_B200_PSTREAM", "1")
        got = alto.cp_apr_mu(t, cfg)
        assert got.inner_iters == ref.inner_iters
        assert_close_rel(got.loglik_trace, ref.loglik_trace, rel=1e-9)
        assert_close_rel(np.asarray(got.kkt_trace), np.asarray(ref.kkt_trace), rel=1e-6)
        assert_close_rel(got.model.weights, ref.model.weights, rel=1e-9)
        for a, b in zip(got.model.factors, ref.model.factors):
            assert_close_rel(a, b, rel=1e-9)


def test_device_als_sweep_matches_host_path(monkeypatch):
    """The device-resident CP-ALS update (Cholesky + triangular solves +
    norms + Grams on the GPU, sweeps replayed as a CUDA graph) against the
    host-solve path, and its fallback to the pseudo-inverse when the normal
    equations are singular (duplicate initial columns)."""
    rng = np.random.default_rng(21)
    dims = (30, 25, 40)
    coords, vals = random_sparse(rng, dims, 3000, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    cfg = alto.CpAlsConfig(rank=6, max_iters=8, fit_tol=1e-300, seed=4)
    monkeypatch.setenv("ALTO_B200_KERNEL", "dview")
    dev = alto.cp_als(t, cfg)
    monkeypatch.setenv("ALTO_B200_HOST_ALS", "1")
    host = alto.cp_als(t, cfg)
    monkeypatch.delenv("ALTO_B200_HOST_ALS")
    assert_close_rel(dev.fit_trace, host.fit_trace, rel=1e-9)
    assert_close_rel(dev.model.weights, host.model.weights, rel=1e-9)
    for a, b in zip(dev.model.factors, host.model.factors):
        assert_close_rel(a, b, rel=1e-9)
    # singular Gram chain -> not positive definite -> host pseudo-inverse path.
    # A singular system's trajectory depends on the last bits of every
    # MTTKRP (the eigh cutoff), so the two runs must execute the same
    # kernels: the plain (non-memoised) deterministic sweep
    base = alto.init_factors(t.shape, 3, seed=1)
    fs = [np.concatenate([f[:, :2], f[:, :1]], axis=1) for f in base.factors]
    init = alto.KruskalModel(np.ones(3), fs)
    cfg3 = alto.CpAlsConfig(rank=3, max_iters=3, fit_tol=1e-300, seed=1)
    monkeypatch.setenv("ALTO_B200_MEMO", "0")
    alto.set_deterministic(True)
    try:
        dsing = alto.cp_als(alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False), cfg3, init=init)
        monkeypatch.setenv("ALTO_B200_HOST_ALS", "1")
        hsing = alto.cp_als(alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False), cfg3, init=init)
    finally:
        alto.set_deterministic(False)
    assert_close_rel(dsing.fit_trace, hsing.fit_trace, rel=1e-9)
    for a, b in zip(dsing.model.factors, hsing.model.factors):
        assert_close_rel(a, b, rel=1e-9, scale=1.0)


@pytest.mark.parametrize("rank", [1, 4, 9, 17, 32, 33])
def test_device_als_update_all_rank_tiles(monkeypatch, rank):
    """Device ALS update for every padded rank tile (4/8/16/32; 33 takes
    the host path) against the host-solve path, on a 4-mode tensor."""
    rng = np.random.default_rng(100 + rank)
    dims = (23, 31, 17, 40)
    coords, vals = random_sparse(rng, dims, 4000, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    cfg = alto.CpAlsConfig(rank=rank, max_iters=4, fit_tol=1e-300, seed=rank)
    dev = alto.cp_als(t, cfg)
    monkeypatch.setenv("ALTO_B200_HOST_ALS", "1")
    host = alto.cp_als(t, cfg)
    assert_close_rel(dev.fit_trace, host.fit_trace, rel=1e-9)
    for a, b in zip(dev.model.factors, host.model.factors):
        assert_close_rel(a, b, rel=1e-8)


@pytest.mark.parametrize("rank", [3, 10, 16, 40])
def test_memoised_sweep_matches_plain_sweep(monkeypatch, rank):
    """Memoised CP-ALS sweep (modes 0 and 1 share sum_k v A_2[k] per (i, j)
    piece, paper_2403_06348_b200/memo.py): MTTKRP outputs of both modes equal
    the oracle to 1e-12, and the CP-ALS trace/factors equal the plain
    decoded-view sweep to 1e-9, on a skewed tensor (long fibers, fibers cut by
    segment edges, rows spanning segments), through the graph sweep."""
    from oracle import alto_oracle as orc
    from paper_2403_06348_b200.cpd import als as ALS

    monkeypatch.setenv("ALTO_B200_KERNEL", "dview")
    rng = np.random.default_rng(300 + rank)
    dims = (60, 150, 3000)
    zipf = [np.minimum(rng.zipf(1.3, 200_000) - 1, d - 1) for d in dims]
    coords = np.unique(np.stack(zipf, axis=1), axis=0)
    vals = rng.random(len(coords)) + 0.1
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    cfg = alto.CpAlsConfig(rank=rank, max_iters=4, fit_tol=1e-300, seed=4)
    st = ALS.AlsState(t, cfg, memo=True)
    assert st._memo() is not None and st._memo().P < t.nnz
    factors = [m[:, :rank].cpu().numpy() for m in st.dfac.mats]
    m0 = st.mttkrp(0).cpu().numpy()
    assert_close_rel(m0, orc.mttkrp(scoords, svals, factors, 0), rel=1e-12)
    m1 = st.mttkrp(1).cpu().numpy()  # same factors: T from the pass above
    assert_close_rel(m1, orc.mttkrp(scoords, svals, factors, 1), rel=1e-12)
    monkeypatch.setenv("ALTO_B200_MEMO", "0")
    ref = alto.cp_als(t, cfg)
    monkeypatch.setenv("ALTO_B200_MEMO", "1")
    got = alto.cp_als(t, cfg)
    assert_close_rel(got.fit_trace, ref.fit_trace, rel=1e-9)
    assert_close_rel(got.model.weights, ref.model.weights, rel=1e-9)
    for a, b in zip(got.model.factors, ref.model.factors):
        assert_close_rel(a, b, rel=1e-9)


@pytest.mark.parametrize("case", ["one_nonzero", "one_row", "one_fiber", "ragged"])
def test_memoised_and_streamed_paths_edge_cases(monkeypatch, case):
    """Degenerate shapes through the memoised CP-ALS sweep and the
    streamed-Pi CP-APR loop: a single nonzero, every nonzero in one output
    row, one (i, j) fiber, and a ragged count just over a segment boundary;
    traces equal the plain paths (1e-9) with identical inner counts."""
    rng = np.random.default_rng(44)
    if case == "one_nonzero":
        dims, coords = (3, 4, 5), np.array([[1, 2, 3]])
    elif case == "one_row":
        dims = (4, 30, 40)
        coords = np.unique(np.stack([np.full(600, 2), rng.integers(0, 30, 600), rng.integers(0, 40, 600)], 1), axis=0)
    elif case == "one_fiber":
        dims = (5, 6, 900)
        coords = np.stack([np.full(700, 3), np.full(700, 4), rng.permutation(900)[:700]], 1)
    else:
        dims = (37, 41, 43)
        coords = np.unique(np.stack([rng.integers(0, d, 700) for d in dims], 1), axis=0)[:513]
    vals = 1.0 + rng.poisson(2.0, len(coords)).astype(np.float64)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    monkeypatch.setenv("ALTO_B200_KERNEL", "dview")
    for flag in ("MEMO", "PSTREAM"):
        monkeypatch.setenv(f"ALTO_B200_{flag}", "0")
    als_ref = alto.cp_als(t, alto.CpAlsConfig(rank=3, max_iters=4, fit_tol=1e-300, seed=1))
    apr_ref = alto.cp_apr_mu(t, alto.CpAprConfig(rank=2, max_outer=3, seed=1))
    for flag in ("MEMO", "PSTREAM"):
        monkeypatch.setenv(f"ALTO_B200_{flag}", "1")
    als = alto.cp_als(t, alto.CpAlsConfig(rank=3, max_iters=4, fit_tol=1e-300, seed=1))
    apr = alto.cp_apr_mu(t, alto.CpAprConfig(rank=2, max_outer=3, seed=1))
    assert_close_rel(als.fit_trace, als_ref.fit_trace, rel=1e-9)
    for a, b in zip(als.model.factors, als_ref.model.factors):
        assert_close_rel(a, b, rel=1e-9)
    assert apr.inner_iters == apr_ref.inner_iters
    assert_close_rel(apr.loglik_trace, apr_ref.loglik_trace, rel=1e-9)
    for a, b in zip(apr.model.factors, apr_ref.model.factors):
        assert_close_rel(a, b, rel=1e-9)
