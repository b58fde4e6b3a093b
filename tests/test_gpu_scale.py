"""BASELINE-config parity: bounded samples of every config against the CPU
oracle (exact keys, 1e-12 fp64), and size-independent properties at the
full c2 size (76M nonzeros): sortedness, cross-kernel agreement, exact
linearity, determinism of the exact output-oriented kernel."""

import numpy as np
import pytest
import torch

import paper_2403_06348_b200 as alto
from conftest import assert_close_rel
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import kernels as K
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.cpd import apr as A

pytestmark = pytest.mark.gpu

SAMPLES = {"c1": 200_000, "c2": 400_000, "c3": 300_000, "c4": 300_000, "c5": 200_000}


@pytest.mark.parametrize("name", sorted(SAMPLES))
def test_config_samples_against_oracle(name):
    cfg = synthetic.CONFIGS[name]
    coords, vals = synthetic.generate_numpy(cfg, SAMPLES[name], seed=5)
    t = alto.AltoTensor.from_coo(alto.CooTensor(cfg.dims, coords, vals))
    keys, svals, scoords = orc.from_coo(cfg.dims, coords, vals)
    assert t.layout.word_bits == (64 if t.layout.total_bits <= 64 else 128)
    assert np.array_equal(t.positions, keys)
    assert np.array_equal(t.values, svals)
    rng = np.random.default_rng(7)
    R = cfg.rank
    factors = [rng.random((d, R)) for d in cfg.dims]
    d = K.DeviceFactors(factors, R)
    for mode in range(len(cfg.dims)):
        want = orc.mttkrp(scoords, svals, factors, mode)
        for kernel in ("dview", "oriented", "atomic"):
            got = K.launch_mttkrp(t, d, mode, kernel)[:, :R].cpu().numpy()
            assert_close_rel(got, want, rel=1e-12)
        if cfg.values == "poisson1p2" or name == "c2":
            scaled = rng.random((cfg.dims[mode], R)) + 0.01
            pwant = orc.phi(scoords, svals, scaled, factors, mode)
            bd = K.nat.to_device_matrix(scaled)
            for kernel in ("dview", "oriented"):
                pgot = A.launch_phi(t, d, mode, kernel, bd, 1e-10)[:, :R].cpu().numpy()
                assert_close_rel(pgot, pwant, rel=1e-12)


@pytest.fixture(scope="module")
def c2_full():
    cfg = synthetic.CONFIGS["c2"]
    coords, vals = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
    del coords
    yield cfg, t
    del t
    torch.cuda.empty_cache()


def test_c2_full_size_properties(c2_full):
    cfg, t = c2_full
    assert t.nnz == cfg.nnz
    k = t._keys
    assert bool((k[1:] > k[:-1]).all())  # < 2^63: signed order == unsigned
    R = cfg.rank
    g = torch.Generator(device="cuda").manual_seed(3)
    fac = [torch.rand((dd, R), dtype=torch.float64, device="cuda", generator=g) for dd in cfg.dims]
    d = K.DeviceFactors(fac, R)
    for mode in range(3):
        a = K.launch_mttkrp(t, d, mode, "dview")[:, :R].clone()
        b = K.launch_mttkrp(t, d, mode, "atomic")[:, :R].clone()
        scale = float(a.abs().max())
        assert float((a - b).abs().max()) <= 1e-12 * scale  # two independent algorithms agree
    # exact output-oriented kernel: deterministic and exactly linear in the values
    mode = 1
    nseg = K.nat.default_segments(t.nnz)
    e1 = K.launch_mttkrp(t, d, mode, "exact-output", num_segments=nseg)[:, :R].clone()
    e2 = K.launch_mttkrp(t, d, mode, "exact-output", num_segments=nseg)[:, :R].clone()
    assert torch.equal(e1, e2)
    t2 = alto.AltoTensor(t.layout, t._keys, t._vals * 2.0, _validate=False)
    e3 = K.launch_mttkrp(t2, d, mode, "exact-output", num_segments=nseg)[:, :R]
    assert torch.equal(e3, 2.0 * e1)
    fast = K.launch_mttkrp(t, d, mode, "dview")[:, :R]
    assert float((fast - e1).abs().max()) <= 1e-12 * float(e1.abs().max())


def test_c2_full_size_memoised_mttkrp(c2_full):
    """BASELINE configs[1] at full size: the memoised pair (mode 0 storing
    the per-piece partial sums, mode 1 streaming them) agrees with the
    stateless decoded-view kernel to 1e-12, and T is exactly linear."""
    from paper_2403_06348_b200.memo import MemoPlan

    cfg, t = c2_full
    R = cfg.rank
    g = torch.Generator(device="cuda").manual_seed(5)
    fac = [torch.rand((dd, R), dtype=torch.float64, device="cuda", generator=g) for dd in cfg.dims]
    d = K.DeviceFactors(fac, R)
    plan = MemoPlan(t, R)
    assert 0 < plan.P < t.nnz
    outs = [torch.zeros((dd, K.nat.padded_ld(R)), dtype=torch.float64, device="cuda") for dd in cfg.dims[:2]]
    plan.mttkrp_m0(t, d, outs[0])
    plan.mttkrp_m1(d, outs[1])
    for mode in (0, 1):
        want = K.launch_mttkrp(t, d, mode, "dview")[:, :R]
        got = outs[mode][:, :R]
        assert float((got - want).abs().max()) <= 1e-12 * float(want.abs().max())
    del plan
    torch.cuda.empty_cache()


def test_c4_full_size_streamed_phi():
    """BASELINE configs[3] at full size: Phi from the stored Khatri-Rao rows
    equals the gathering Phi to 1e-12 for every mode, and the streamed
    log-likelihood equals the gathering one."""
    cfg = synthetic.CONFIGS["c4"]
    coords, vals = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
    del coords, vals
    R = cfg.rank
    g = torch.Generator(device="cuda").manual_seed(6)
    d = K.DeviceFactors([torch.rand((dd, R), dtype=torch.float64, device="cuda", generator=g) for dd in cfg.dims], R)
    w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g) + 0.5
    pil = torch.empty(A.pstream_sizes(t, R)[1], dtype=torch.float64, device="cuda")
    for mode in range(3):
        b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda", generator=g)
        gat = A.launch_phi(t, d, mode, "dview", b, 1e-10, pi_il_out=pil)[:, :R].clone()
        out = torch.zeros_like(b)
        got = A.launch_phi_pstream(t, mode, R, b, 1e-10, pil, out)[:, :R]
        assert float((got - gat).abs().max()) <= 1e-12 * float(gat.abs().max())
        ll_s = float(A.loglik_data_term_pstream(t, d, w, mode, pil))
        ll_g = float(A.loglik_data_term_dview(t, d, w, mode=mode))
        assert ll_s == pytest.approx(ll_g, rel=1e-12)
    del t, pil
    torch.cuda.empty_cache()
