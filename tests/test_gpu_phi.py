"""Phi (CP-APR model-update ratio), Khatri-Rao rows and the fused KKT
epilogue on the B200 vs the reference (pkg/tests/test_cpd_apr.py)."""

import numpy as np
import pytest
import torch

import paper_2403_06348_b200 as alto
from conftest import (
    EXAMPLE_COORDS,
    EXAMPLE_DIMS,
    EXAMPLE_VALUES,
    assert_close_rel,
    case_factors,
    golden,
    random_cases,
    random_sparse,
)
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import kernels as K
from paper_2403_06348_b200.cpd import apr as A
from paper_2403_06348_b200.partition import dview_order

pytestmark = pytest.mark.gpu


def example():
    return alto.AltoTensor.from_coo(alto.CooTensor(EXAMPLE_DIMS, EXAMPLE_COORDS, EXAMPLE_VALUES))


def _tensor(g):
    dims = tuple(int(x) for x in g["dims"])
    return dims, alto.AltoTensor.from_coo(alto.CooTensor(dims, g["in_coords"], g["in_values"]))


@pytest.mark.parametrize("case", random_cases())
def test_pi_and_exact_phi_bitwise(case):
    g = golden(case)
    dims, t = _tensor(g)
    factors = case_factors(g)
    for mode in range(len(dims)):
        pi = alto.precompute_krp_rows(t, factors, mode)
        assert np.array_equal(pi, g[f"pi_m{mode}"])
        scaled = g[f"scaled_m{mode}"]
        got = alto.phi_kernel(t, scaled, factors, mode, strategy="sequential", exact=True)
        assert np.array_equal(got, g[f"phiseq_m{mode}"])
        pre = alto.phi_kernel(t, scaled, factors, mode, krp_rows=pi, strategy="sequential", exact=True)
        assert np.array_equal(pre, g[f"phiseq_m{mode}"])
        for L in (2, 4, 7):
            rec = alto.phi_kernel(t, scaled, factors, mode, workers=2, num_segments=L,
                                  strategy="recursive", exact=True)
            assert np.array_equal(rec, g[f"phirec{L}_m{mode}"])
            out = alto.phi_kernel(t, scaled, factors, mode, workers=2, num_segments=L,
                                  strategy="output", exact=True)
            assert np.array_equal(out, g[f"phiout{L}_m{mode}"])
            outp = alto.phi_kernel(t, scaled, factors, mode, krp_rows=pi, workers=2, num_segments=L,
                                   strategy="output", exact=True)
            assert np.array_equal(outp, g[f"phiout{L}_m{mode}"])


@pytest.mark.parametrize("case", random_cases())
@pytest.mark.parametrize("kernel", ["dview", "oriented", "atomic"])
def test_fast_phi_close_and_pre_equals_otf(case, kernel):
    g = golden(case)
    dims, t = _tensor(g)
    factors = case_factors(g)
    d = K.DeviceFactors(factors)
    for mode in range(len(dims)):
        b = torch.from_numpy(g[f"scaled_m{mode}"]).cuda()
        bd = K.nat.to_device_matrix(b)
        otf = A.launch_phi(t, d, mode, kernel, bd, 1e-10)[:, : d.rank].cpu().numpy()
        assert_close_rel(otf, g[f"phiseq_m{mode}"], rel=1e-12)
        if kernel in ("oriented", "dview"):
            # PRE rows in the order the kernel walks
            vkeys = (dview_order(t, mode, d.rank) if kernel == "dview" else K.device_mode_view(t, mode))[1]
            pv = A.launch_pi(t, d, mode, keys=vkeys)
            if kernel == "dview":  # the decoded-view builder gives the same rows bit for bit
                assert torch.equal(A.launch_pi_dview(t, d, mode), pv)
            pre = A.launch_phi(t, d, mode, kernel, bd, 1e-10, pi_view=pv)
        else:
            pre = A.launch_phi(t, d, mode, kernel, bd, 1e-10, pi=A.launch_pi(t, d, mode))
        pre = pre[:, : d.rank].cpu().numpy()
        if kernel in ("oriented", "dview"):
            assert np.array_equal(pre, otf)  # same kernel, same multiply order
        else:
            assert_close_rel(pre, otf, rel=1e-12)


def test_exact_model_gives_ones():
    rng = np.random.default_rng(2)
    factors = [rng.dirichlet(np.ones(2), size=1).T for _ in range(3)]
    model = alto.KruskalModel(np.array([8.0]), factors)
    t = alto.AltoTensor.from_coo(alto.CooTensor.from_dense(model.to_dense()))
    for exact in (True, False):
        phi = alto.phi_kernel(t, model.factors[0] * model.weights, model.factors, 0, exact=exact)
        assert_close_rel(phi, np.ones((2, 1)), rel=1e-12, scale=1.0)


def test_eps_clamp():
    t = example()
    factors = [np.ones((d, 1)) for d in EXAMPLE_DIMS]
    for exact in (True, False):
        phi = alto.phi_kernel(t, np.zeros((4, 1)), factors, 0, eps=1e-10, exact=exact)
        assert_close_rel(phi, np.array([[1.0], [5.0], [4.0], [11.0]]) / 1e-10, rel=1e-15)


def test_shape_validation():
    t = example()
    factors = [np.ones((d, 2)) for d in EXAMPLE_DIMS]
    with pytest.raises(ValueError, match="scaled"):
        alto.phi_kernel(t, np.ones((5, 2)), factors, 0)
    with pytest.raises(ValueError, match="krp_rows"):
        alto.phi_kernel(t, np.ones((4, 2)), factors, 0, krp_rows=np.ones((3, 2)))


def test_apr_update_fused_epilogue():
    rng = np.random.default_rng(6)
    b = rng.random((50, 7))
    phi = rng.random((50, 7)) * 2
    want = orc.kkt(b, phi)
    bd = K.nat.to_device_matrix(b)
    pd = K.nat.to_device_matrix(phi)
    kkt, nonfinite = A.apr_update(bd, pd, 7, tau=1e-4, apply=-1)
    assert kkt == want and not nonfinite
    assert np.array_equal(bd[:, :7].cpu().numpy(), b * phi)  # applied: kkt >= tau
    bd2 = K.nat.to_device_matrix(b)
    kkt2, _ = A.apr_update(bd2, K.nat.to_device_matrix(np.ones((50, 7))), 7, tau=1e-4, apply=-1)
    assert kkt2 == 0.0 and np.array_equal(bd2[:, :7].cpu().numpy(), b)  # converged: untouched
    big = K.nat.to_device_matrix(np.full((4, 2), 1e300))
    _, nf = A.apr_update(big, K.nat.to_device_matrix(np.full((4, 2), 1e300)), 2, tau=1e-4, apply=-1)
    assert nf


def test_loglik_matches_oracle():
    rng = np.random.default_rng(9)
    coords, vals = random_sparse(rng, (30, 20, 25), 2000, kind="counts")
    t = alto.AltoTensor.from_coo(alto.CooTensor((30, 20, 25), coords, vals))
    model = alto.init_factors((30, 20, 25), 5, seed=3, nonneg=True).normalized(1)
    got = alto.poisson_loglik(t, model)
    want = orc.loglik(t.coords, t.values, model.weights, model.factors)
    assert got == pytest.approx(want, rel=1e-12)


def test_loglik_decoded_view_matches_key_stream_kernel():
    """The decoded-view log-likelihood (Phi's B-row machinery with
    B = lambda o A_mode) against the key-stream kernel and the oracle."""
    from paper_2403_06348_b200.cpd.apr import loglik_data_term, loglik_data_term_dview

    rng = np.random.default_rng(31)
    for dims, R in (((30, 40, 50), 5), ((20, 30, 25, 12), 10), ((300, 400, 90), 16)):
        coords, vals = random_sparse(rng, dims, 4000, kind="counts")
        t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
        factors = [rng.random((d, R)) + 0.05 for d in dims]
        lam = rng.random(R) + 0.5
        d = K.DeviceFactors(factors, R)
        w = torch.from_numpy(lam).cuda()
        want = loglik_data_term(t, d, w)
        for mode in range(len(dims)):
            got = float(loglik_data_term_dview(t, d, w, mode=mode))
            assert abs(got - want) <= 1e-12 * abs(want)
        model = alto.KruskalModel(lam, factors)
        oracle_data = float(np.sum(t.values * np.log(model.values_at(t.coords))))
        assert abs(want - oracle_data) <= 1e-12 * abs(oracle_data)


@pytest.mark.parametrize("ndim,rank", [(3, 10), (3, 16), (4, 5), (5, 3), (3, 1)])
@pytest.mark.parametrize("block", ["0", "1"])
def test_streamed_pi_phi_matches_otf(monkeypatch, ndim, rank, block):
    """Streamed-Pi Phi (csrc/pstream.cu): the on-the-fly dview Phi stores the
    Khatri-Rao rows in the slot layout while it runs; Phi from those rows
    equals the gathered Phi (and the oracle) to rounding, including ragged
    last segments, runs crossing 128-nonzero chunks and blocked views."""
    monkeypatch.setenv("ALTO_B200_BLOCK", block)
    monkeypatch.setenv("ALTO_B200_BLOCK_MIN_RUN", "0")
    rng = np.random.default_rng(500 + 7 * ndim + rank)
    dims = {3: (37, 900, 1300), 4: (30, 40, 50, 60), 5: (9, 10, 11, 12, 13)}[ndim]
    coords, vals = random_sparse(rng, dims, 40_001, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    slots, pid = A.pstream_sizes(t, rank)
    assert slots % (512 * 32) == 0 and slots >= t.nnz and pid == slots * rank
    pil = torch.full((pid,), float("nan"), dtype=torch.float64, device="cuda")
    for mode in range(ndim):
        scaled = rng.random((dims[mode], rank)) + 0.01
        bd = K.nat.to_device_matrix(scaled)
        otf = A.launch_phi(t, d, mode, "dview", bd, 1e-10, pi_il_out=pil)[:, :rank].cpu().numpy()
        out = torch.zeros((dims[mode], K.nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
        got = A.launch_phi_pstream(t, mode, rank, bd, 1e-10, pil, out)[:, :rank].cpu().numpy()
        want = orc.phi(scoords, svals, scaled, factors, mode)
        assert_close_rel(got, otf, rel=1e-12)
        assert_close_rel(got, want, rel=1e-12)


@pytest.mark.parametrize("ndim,rank", [(3, 10), (4, 5), (3, 16)])
def test_streamed_pi_loglik_matches_gathering(ndim, rank):
    """Log-likelihood data term from the stored Khatri-Rao rows of a mode
    (csrc/pstream.cu, LL) equals the gathering decoded-view kernel and the
    oracle's sum v log(mhat)."""
    rng = np.random.default_rng(900 + ndim + rank)
    dims = {3: (41, 700, 1200), 4: (30, 40, 50, 60)}[ndim]
    coords, vals = random_sparse(rng, dims, 30_007, kind="counts")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    factors = [rng.random((d, rank)) + 0.05 for d in dims]
    weights = rng.random(rank) + 0.5
    d = K.DeviceFactors(factors, rank)
    w = torch.from_numpy(weights).cuda()
    _slots, pid = A.pstream_sizes(t, rank)
    pil = torch.empty(pid, dtype=torch.float64, device="cuda")
    mhat = alto.KruskalModel(weights, factors).values_at(t.coords) if hasattr(alto.KruskalModel, "values_at") else None
    for mode in range(ndim):
        b = torch.rand((dims[mode], K.nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
        A.launch_phi(t, d, mode, "dview", b, 1e-10, pi_il_out=pil)
        got = float(A.loglik_data_term_pstream(t, d, w, mode, pil))
        ref = float(A.loglik_data_term_dview(t, d, w, mode=mode))
        assert got == pytest.approx(ref, rel=1e-12)
        if mhat is not None:
            assert got == pytest.approx(float(np.sum(t.values * np.log(mhat))), rel=1e-11)


@pytest.mark.parametrize("rank", [10, 3, 16])
def test_streamed_pi_compact_layout_bitwise(monkeypatch, rank):
    """Count data with < 65536 rows per mode streams u16 rows and u8 values
    (csrc/pstream.cu CMP): Phi and the log-likelihood equal the u32 / f64
    layout's to rounding (the same arithmetic per nonzero; runs cut by chunk
    edges are fp64 reductions in either layout, so not run-to-run bitwise);
    values above 255 or non-integral keep the full layout."""
    rng = np.random.default_rng(1300 + rank)
    dims = (41, 700, 1200)
    coords, vals = random_sparse(rng, dims, 30_011, kind="counts")
    factors = [rng.random((d, rank)) + 0.05 for d in dims]
    d = K.DeviceFactors(factors, rank)
    w = torch.from_numpy(rng.random(rank) + 0.5).cuda()
    _slots, pid = A.pstream_sizes(alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals)), rank)
    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("ALTO_B200_PSTREAM_COMPACT", flag)
        t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
        pil = torch.empty(pid, dtype=torch.float64, device="cuda")
        outs = []
        for mode in range(3):
            b = torch.from_numpy(np.random.default_rng(mode).random((dims[mode], K.nat.padded_ld(rank)))).cuda()
            A.launch_phi(t, d, mode, "dview", b, 1e-10, pi_il_out=pil)
            assert A.pstream_view(t, mode, rank)[2] == (flag == "1")
            out = torch.zeros((dims[mode], K.nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
            outs.append(A.launch_phi_pstream(t, mode, rank, b, 1e-10, pil, out)[:, :rank].cpu().numpy())
            outs.append(float(A.loglik_data_term_pstream(t, d, w, mode, pil)))
        res[flag] = outs
    for a, b in zip(res["1"], res["0"]):
        assert_close_rel(np.atleast_1d(a), np.atleast_1d(b), rel=1e-13)
    big = vals.copy()
    big[0] = 300.0
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, big))
    monkeypatch.setenv("ALTO_B200_PSTREAM_COMPACT", "1")
    assert A.pstream_view(t, 0, rank)[2] is False
