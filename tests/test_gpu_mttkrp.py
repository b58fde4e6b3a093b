"""MTTKRP on the B200 vs the reference.

exact=True: every strategy must be BIT-IDENTICAL to the reference's output
for the same segment count (golden fixtures). Fast kernels: within 1e-12
relative of the reference (fp64; north_star tolerance is 1e-9)."""

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
    dense_mttkrp_oracle,
    golden,
    random_cases,
    random_sparse,
)
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _tensor(g):
    dims = tuple(int(x) for x in g["dims"])
    return dims, alto.AltoTensor.from_coo(alto.CooTensor(dims, g["in_coords"], g["in_values"]))


def example():
    return alto.AltoTensor.from_coo(alto.CooTensor(EXAMPLE_DIMS, EXAMPLE_COORDS, EXAMPLE_VALUES))


def ones(dims, rank=1):
    return [np.ones((d, rank)) for d in dims]


class TestWorkedExample:
    @pytest.mark.parametrize("exact", [True, False])
    def test_all_strategies_ones(self, exact):
        t = example()
        assert alto.mttkrp_sequential(t, ones(EXAMPLE_DIMS), 0, exact=exact).ravel().tolist() == [1, 5, 4, 11]
        segs = alto.make_segments(t, 2)
        out = alto.mttkrp_recursive(t, segs, ones(EXAMPLE_DIMS), 0, 2, exact=exact)
        assert out.ravel().tolist() == [1, 5, 4, 11]
        view = alto.make_mode_ordered_view(t, 0, 2)
        out = alto.mttkrp_output_oriented(t, view, ones(EXAMPLE_DIMS), 0, 2, exact=exact)
        assert out.ravel().tolist() == [1, 5, 4, 11]

    @pytest.mark.parametrize("kernel", ["dview", "oriented", "atomic", "segment", "segment-atomic",
                                        "exact-seq", "exact-rec", "exact-output"])
    def test_every_gpu_kernel(self, kernel):
        t = example()
        d = K.DeviceFactors(ones(EXAMPLE_DIMS), 1)
        out = K.launch_mttkrp(t, d, 0, kernel, num_segments=2)[:, :1].cpu().numpy()
        assert out.ravel().tolist() == [1, 5, 4, 11]

    def test_empty_row_stays_zero(self):
        t = alto.AltoTensor.from_coo(alto.CooTensor((3, 2), [[0, 0], [2, 1]], [1.0, 2.0]))
        for exact in (True, False):
            assert alto.mttkrp_sequential(t, ones((3, 2)), 0, exact=exact).ravel().tolist() == [1, 0, 2]

    def test_contended_single_row(self):
        t = alto.AltoTensor.from_coo(alto.CooTensor((2, 8), [[1, j] for j in range(8)], np.ones(8)))
        f = [np.ones((2, 3)), np.ones((8, 3))]
        for exact in (True, False):
            view = alto.make_mode_ordered_view(t, 0, 4)
            out = alto.mttkrp_output_oriented(t, view, f, 0, 4, exact=exact)
            assert out[1].tolist() == [8.0, 8.0, 8.0] and out[0].tolist() == [0.0, 0.0, 0.0]
            assert alto.mttkrp(t, f, 0, exact=exact)[1].tolist() == [8.0, 8.0, 8.0]


@pytest.mark.parametrize("case", random_cases())
def test_exact_strategies_bitwise(case):
    g = golden(case)
    dims, t = _tensor(g)
    factors = case_factors(g)
    for mode in range(len(dims)):
        got = alto.mttkrp_sequential(t, factors, mode, exact=True)
        assert np.array_equal(got, g[f"seq_m{mode}"]), f"sequential mode {mode}"
        for L in (2, 4, 7):
            segs = alto.make_segments(t, L)
            got = alto.mttkrp_recursive(t, segs, factors, mode, 2, exact=True)
            assert np.array_equal(got, g[f"rec{L}_m{mode}"]), f"recursive L={L} mode {mode}"
            view = alto.make_mode_ordered_view(t, mode, L)
            got = alto.mttkrp_output_oriented(t, view, factors, mode, 2, exact=True)
            assert np.array_equal(got, g[f"out{L}_m{mode}"]), f"output L={L} mode {mode}"


@pytest.mark.parametrize("case", random_cases())
@pytest.mark.parametrize("kernel", ["dview", "oriented", "atomic", "segment", "segment-atomic"])
def test_fast_kernels_close(case, kernel):
    g = golden(case)
    dims, t = _tensor(g)
    factors = case_factors(g)
    d = K.DeviceFactors(factors)
    for mode in range(len(dims)):
        got = K.launch_mttkrp(t, d, mode, kernel)[:, : d.rank].cpu().numpy()
        assert_close_rel(got, g[f"seq_m{mode}"], rel=1e-12)


def test_dense_oracle_many_shapes():
    """Acceptance-#3-style sweep: N in {3,4,5}, R in {1,2,8,16}, all kernels
    against the dense matricised oracle at 1e-12 (pkg/tests/test_acceptance.py:124-153)."""
    rng = np.random.default_rng(3)
    ranks = [1, 2, 8, 16]
    for trial in range(40):
        ndim = int(rng.integers(3, 6))
        dims = tuple(int(d) for d in rng.integers(2, 21, size=ndim))
        coords, vals = random_sparse(rng, dims, int(rng.integers(10, 501)), kind="positive")
        coo = alto.CooTensor(dims, coords, vals)
        t = alto.AltoTensor.from_coo(coo)
        rank = ranks[trial % 4]
        factors = [rng.random((d, rank)) + 0.05 for d in dims]
        mode = int(rng.integers(0, ndim))
        want = dense_mttkrp_oracle(coo.to_dense(), factors, mode)
        tol = 1e-12 * np.maximum(np.abs(want), np.abs(want).max() * 1e-6 + 1e-300)
        for strategy in ("sequential", "recursive", "output"):
            for exact in (True, False):
                got = alto.mttkrp(t, factors, mode, workers=2, num_segments=4, strategy=strategy, exact=exact)
                assert (np.abs(got - want) <= tol).all(), (trial, strategy, exact)


def test_wide_128bit():
    g = golden("wide128")
    dims = tuple(int(x) for x in g["dims"])
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, g["in_coords"], g["in_values"]))
    factors = [np.random.default_rng(int(s)).random((d, 4)) for s, d in zip(g["factor_seeds"], dims)]
    for mode in range(4):
        rows = g[f"seq_m{mode}_rows"]
        exact = alto.mttkrp_sequential(t, factors, mode, exact=True)
        assert np.array_equal(exact[rows], g[f"seq_m{mode}_vals"])
        fast = alto.mttkrp(t, factors, mode)
        assert_close_rel(fast[rows], g[f"seq_m{mode}_vals"], rel=1e-12)


@pytest.mark.parametrize("ndim,rank", [(2, 3), (6, 5), (7, 12), (3, 40), (4, 33)])
def test_generic_modes_and_wide_ranks(ndim, rank):
    """Mode counts outside the specialised kernels and ranks > 32 (rank
    chunking) against the oracle's sequential kernel."""
    rng = np.random.default_rng(ndim * 100 + rank)
    dims = tuple(int(d) for d in rng.integers(3, 12, size=ndim))
    coords, vals = random_sparse(rng, dims, 400, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    factors = [rng.random((d, rank)) for d in dims]
    for mode in range(ndim):
        want = orc.mttkrp(t.coords, t.values, factors, mode)
        assert np.array_equal(alto.mttkrp_sequential(t, factors, mode, exact=True), want)
        for kernel in (("dview",) if ndim <= 5 else ()) + ("oriented", "atomic"):
            got = K.launch_mttkrp(t, K.DeviceFactors(factors), mode, kernel)[:, :rank].cpu().numpy()
            assert_close_rel(got, want, rel=1e-12)


class TestDeterminismAndApi:
    def test_exact_recursive_repeatable(self):
        rng = np.random.default_rng(31)
        coords, vals = random_sparse(rng, (9, 7, 8), 150)
        t = alto.AltoTensor.from_coo(alto.CooTensor((9, 7, 8), coords, vals))
        factors = [rng.random((d, 8)) for d in (9, 7, 8)]
        runs = [alto.mttkrp(t, factors, 0, workers=w, num_segments=5, strategy="recursive", exact=True)
                for w in (1, 2, 4, 7)]
        for r in runs[1:]:
            assert (r == runs[0]).all()

    def test_exact_output_deterministic_many_segments(self):
        rng = np.random.default_rng(32)
        coords, vals = random_sparse(rng, (50, 40, 60), 5000)
        t = alto.AltoTensor.from_coo(alto.CooTensor((50, 40, 60), coords, vals))
        factors = [rng.random((d, 16)) for d in (50, 40, 60)]
        d = K.DeviceFactors(factors)
        a = K.launch_mttkrp(t, d, 1, "exact-output", num_segments=977).cpu().numpy()
        b = K.launch_mttkrp(t, d, 1, "exact-output", num_segments=977).cpu().numpy()
        assert (a == b).all()
        want = orc.mttkrp(t.coords, t.values, factors, 1, "output", 977)
        assert np.array_equal(a[:, :16], want)

    def test_torch_in_torch_out(self):
        t = example()
        f = [torch.ones((d, 2), dtype=torch.float64, device="cuda") for d in EXAMPLE_DIMS]
        out = alto.mttkrp(t, f, 0)
        assert isinstance(out, torch.Tensor) and out.is_cuda
        assert out[:, 0].cpu().tolist() == [1, 5, 4, 11]

    def test_validation_messages(self):
        t = example()
        with pytest.raises(ValueError, match="rows"):
            alto.mttkrp(t, [np.ones((5, 2)), np.ones((8, 2)), np.ones((2, 2))], 0)
        with pytest.raises(ValueError, match="columns"):
            alto.mttkrp(t, [np.ones((4, 2)), np.ones((8, 3)), np.ones((2, 2))], 0)
        with pytest.raises(ValueError, match="mode"):
            alto.mttkrp(t, ones(EXAMPLE_DIMS), 5)
        bad = ones(EXAMPLE_DIMS)
        bad[1][3, 0] = np.nan
        with pytest.raises(ValueError, match="finite"):
            alto.mttkrp(t, bad, 0)
        # the scan is deferred to the result read-back: the lowest bad mode is
        # named, including the target mode's factor (checked on the host)
        for bad_modes, target, named in (((1, 2), 0, 1), ((0, 2), 0, 0), ((2,), 1, 2), ((0,), 0, 0)):
            bad = ones(EXAMPLE_DIMS)
            for m in bad_modes:
                bad[m][-1, 0] = np.inf if m % 2 else np.nan
            with pytest.raises(ValueError, match=f"factor {named} contains non-finite"):
                alto.mttkrp(t, bad, target)
            with pytest.raises(ValueError, match=f"factor {named} contains non-finite"):
                alto.mttkrp_sequential(t, bad, target)
        big = ones(EXAMPLE_DIMS)
        big[0][:] = 1e308  # the host sum overflows but every entry is finite
        alto.mttkrp(t, big, 0)  # no error: overflowed sums fall back to the exact scan
        alto.mttkrp(t, big, 1)
        with pytest.raises(ValueError, match="strategy"):
            alto.mttkrp(t, ones(EXAMPLE_DIMS), 0, strategy="fastest")

    def test_choice_records(self):
        t = example()
        _, c = K.mttkrp_with_choice(t, ones(EXAMPLE_DIMS, 2), 0, workers=2)
        assert c.strategy is alto.Strategy.OUTPUT_ORIENTED  # reuse 1.5, like the reference
        _, c = K.mttkrp_with_choice(t, ones(EXAMPLE_DIMS), 0)
        assert c.strategy is alto.Strategy.SEQUENTIAL
        _, c = K.mttkrp_with_choice(t, ones(EXAMPLE_DIMS), 0, workers=2, strategy="recursive")
        assert c.strategy is alto.Strategy.RECURSIVE and c.reason == "explicit request"
        assert c.kernel in K.GPU_KERNELS


def test_blocked_fiber_view_matches_oracle(monkeypatch):
    """Blocked decoded views (rows recur once per block of the largest other
    mode; every run reduced) against the oracle, MTTKRP and Phi, PRE == OTF."""
    from paper_2403_06348_b200.cpd import apr as A
    from paper_2403_06348_b200.partition import dview_order, view_plan

    monkeypatch.setenv("ALTO_B200_BLOCK_MIN_RUN", "0")
    rng = np.random.default_rng(77)
    dims = (40, 1500, 2600)
    coords, vals = random_sparse(rng, dims, 60_000, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    keys, svals, scoords = orc.from_coo(dims, coords, vals)
    R = 16
    factors = [rng.random((d, R)) for d in dims]
    d = K.DeviceFactors(factors, R)
    for mode in range(3):
        fm, bmode, shift = view_plan(t, mode, R)
        assert bmode >= 0 and shift == 9  # 512-row blocks of the largest other mode
        got = K.launch_mttkrp(t, d, mode, "dview")[:, :R].cpu().numpy()
        assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)
        scaled = rng.random((dims[mode], R)) + 0.01
        bd = K.nat.to_device_matrix(scaled)
        otf = A.launch_phi(t, d, mode, "dview", bd, 1e-10)[:, :R].cpu().numpy()
        assert_close_rel(otf, orc.phi(scoords, svals, scaled, factors, mode), rel=1e-12)
        pre = A.launch_phi(t, d, mode, "dview", bd, 1e-10,
                           pi_view=A.launch_pi(t, d, mode, keys=dview_order(t, mode, R)[1]))
        assert_close_rel(pre[:, :R].cpu().numpy(), otf, rel=1e-12)  # same order; atomics reorder runs


@pytest.mark.parametrize("block", ["0", "1"])
@pytest.mark.parametrize("order", ["short", "long"])
@pytest.mark.parametrize("rank", [10, 16, 32])
def test_dview_view_orders_match_oracle(monkeypatch, block, order, rank):
    """Decoded-view MTTKRP and Phi against the oracle over unblocked and
    blocked views, with either fiber sub-order; skewed coordinates so that
    fibers are long and cross segment edges."""
    from paper_2403_06348_b200.cpd import apr as A

    monkeypatch.setenv("ALTO_B200_BLOCK", block)
    monkeypatch.setenv("ALTO_B200_BLOCK_MIN_RUN", "0")
    monkeypatch.setenv("ALTO_B200_FIBER_ORDER", order)
    rng = np.random.default_rng(91 + rank)
    dims = (30, 700, 2600)
    M = 50_000
    zipf = [np.minimum(rng.zipf(1.3, 4 * M) - 1, d - 1) for d in dims]
    coords = np.unique(np.stack(zipf, axis=1), axis=0)
    coords = coords[rng.permutation(len(coords))[:M]]
    vals = rng.random(len(coords)) + 0.5
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    for mode in range(3):
        got = K.launch_mttkrp(t, d, mode, "dview")[:, :rank].cpu().numpy()
        assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)
        scaled = rng.random((dims[mode], rank)) + 0.01
        bd = K.nat.to_device_matrix(scaled)
        phi = A.launch_phi(t, d, mode, "dview", bd, 1e-10)[:, :rank].cpu().numpy()
        assert_close_rel(phi, orc.phi(scoords, svals, scaled, factors, mode), rel=1e-12)


@pytest.mark.parametrize("rank", [1, 5, 16, 32, 40])
@pytest.mark.parametrize("kernel", ["segment", "segment-atomic"])
def test_segment_kernel_hot_rows_and_tiles(rank, kernel):
    """The ALTO line-segment kernel (csrc/segment.cu) on a tensor whose short
    mode has a hot row holding half the nonzeros: segments span many tiles,
    rows cross the group chunks of the row-ordered tile (owner chains), and
    rank > 32 runs in column chunks. Against the oracle, 1e-12 relative."""
    rng = np.random.default_rng(rank)
    dims = (50, 3000, 4000, 7)
    M = 600_000
    hot = rng.random(M) < 0.5
    c0 = np.where(hot, 0, rng.integers(0, dims[0], M))
    coords = np.stack([c0] + [rng.integers(0, d, M) for d in dims[1:]], axis=1)
    vals = rng.random(M) + 0.1
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    keys, svals, scoords = orc.from_coo(dims, *orc.canonicalize(coords, vals))
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    for mode in range(len(dims)):
        plan = K.segment_plan(t, mode, rank)
        if kernel == "segment" and plan["smem_bytes"] > 227 * 1024:
            continue  # interval too wide for shared memory (the heuristic never picks it)
        got = K.launch_mttkrp(t, d, mode, kernel)[:, :rank].cpu().numpy()
        want = orc.mttkrp(scoords, svals, factors, mode)
        assert_close_rel(got, want, rel=1e-12)


def test_gpu_kernel_choice_follows_measured_ranking(monkeypatch):
    """select_gpu_kernel: decoded view while it fits in device memory; else
    the ALTO segment kernel where the widest segment interval fits in shared
    memory (short, high-reuse modes); else direct atomics. The choice and
    its reason are recorded in StrategyChoice (kernel, kernel_reason)."""
    rng = np.random.default_rng(4)
    dims = (40, 5000, 7000)
    coords = np.stack([rng.integers(0, d, 200_000) for d in dims], axis=1)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, rng.random(200_000) + 0.1))
    kern, why = K.select_gpu_kernel(t, 0, 16, None)
    assert kern == "dview" and "fits" in why
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda *a, **k: (1 << 20, 1 << 30))
    kern, why = K.select_gpu_kernel(t, 0, 16, None)
    assert kern == "segment" and "fiber reuse" in why, why
    kern, why = K.select_gpu_kernel(t, 2, 16, None)
    assert kern == "atomic", why
    factors = [rng.random((d, 16)) for d in dims]
    out, choice = K.mttkrp_with_choice(t, factors, 0)
    assert choice.kernel == "segment"
    want = orc.mttkrp(t.coords, t.values, factors, 0)
    assert_close_rel(out, want, rel=1e-12)

