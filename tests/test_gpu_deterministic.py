"""Deterministic mode (csrc/det.cu): the fast decoded-view kernels and the
memoised CP-ALS sweep park segment-edge runs and fold them in a fixed order
instead of fp64 reductions, so repeated runs are bitwise identical (the
reference's bitwise tests: pkg/tests/test_kernels.py:94-114,
test_cpd_apr.py:189-214), and still match the oracle to 1e-12."""

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


@pytest.fixture
def det():
    alto.set_deterministic(True)
    yield
    alto.set_deterministic(False)


def _hot_tensor(seed=0, M=300_000):
    """Zipf coordinates: hot rows span thousands of 512-nonzero segments."""
    rng = np.random.default_rng(seed)
    dims = (90, 700, 2600)
    zipf = [np.minimum(rng.zipf(1.25, 3 * M) - 1, d - 1) for d in dims]
    coords = np.unique(np.stack(zipf, axis=1), axis=0)
    coords = coords[rng.permutation(len(coords))[:M]]
    vals = rng.random(len(coords)) + 0.5
    return dims, coords, vals


@pytest.mark.parametrize("rank", [10, 16, 40])
def test_det_kernels_bitwise_repeatable_and_close(det, monkeypatch, rank):
    monkeypatch.setenv("ALTO_B200_BLOCK_MIN_RUN", "0")  # would block the views without det
    dims, coords, vals = _hot_tensor(rank)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _k, svals, scoords = orc.from_coo(dims, coords, vals)
    rng = np.random.default_rng(1)
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    for mode in range(3):
        a = K.launch_mttkrp(t, d, mode, "dview")[:, :rank].clone()
        b = K.launch_mttkrp(t, d, mode, "dview")[:, :rank].clone()
        assert torch.equal(a, b)
        assert not t._cache[("dview", mode)][4]  # unblocked (no run-wide atomics)
        assert_close_rel(a.cpu().numpy(), orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)
        if rank <= 32:
            scaled = rng.random((dims[mode], rank)) + 0.01
            bd = K.nat.to_device_matrix(scaled)
            p1 = A.launch_phi(t, d, mode, "dview", bd, 1e-10)[:, :rank].clone()
            p2 = A.launch_phi(t, d, mode, "dview", bd, 1e-10)[:, :rank].clone()
            assert torch.equal(p1, p2)
            assert_close_rel(p1.cpu().numpy(), orc.phi(scoords, svals, scaled, factors, mode), rel=1e-12)


def test_det_memoised_cp_als_bitwise_repeatable(det):
    dims, coords, vals = _hot_tensor(7)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    cfg = alto.CpAlsConfig(rank=16, max_iters=5, fit_tol=1e-300, seed=2)
    r1 = alto.cp_als(t, cfg)
    r2 = alto.cp_als(alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False), cfg)
    assert r1.fit_trace == r2.fit_trace
    assert np.array_equal(r1.model.weights, r2.model.weights)
    for a, b in zip(r1.model.factors, r2.model.factors):
        assert np.array_equal(a, b)
    _k, svals, scoords = orc.from_coo(dims, coords, vals)
    _w, _f, fits = orc.cp_als(dims, scoords, svals, 16, 5, seed=2)
    assert_close_rel(r1.fit_trace, fits, rel=1e-9)


def test_det_c2_full_size_sweeps_bitwise_repeatable(det):
    """BASELINE configs[1] at full size: two independent CP-ALS runs of 4
    sweeps (memoised pairs + device update, graph replay) are bitwise equal."""
    cfg = synthetic.CONFIGS["c2"]
    c, v = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
    del c, v
    als = alto.CpAlsConfig(rank=16, max_iters=4, fit_tol=1e-300, seed=0)
    r1 = alto.cp_als(t, als)
    r2 = alto.cp_als(alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False), als)
    assert r1.fit_trace == r2.fit_trace
    for a, b in zip(r1.model.factors, r2.model.factors):
        assert np.array_equal(a, b)
    del t
    torch.cuda.empty_cache()
