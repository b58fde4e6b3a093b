"""Kernels over interleaved (bulk-copy staged) fiber streams against the
oracle: the public 3-mode MTTKRP through the fused fiber kernel, the
memoised sweep's producers (fused branch-free kernel and memo0, which must
write the same T rows bit for bit) and the streaming consumer.
Reference semantics: pkg/src/alto/kernels.py:160-166 (MTTKRP),
pkg/src/alto/cpd/als.py:84-96 (the sweep the memo serves)."""


import numpy as np
import pytest
import torch

import paper_2403_06348_b200 as alto
from conftest import assert_close_rel
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import _native as nat
from paper_2403_06348_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _skewed(seed, dims, draws, alpha=1.3, take=None):
    rng = np.random.default_rng(seed)
    zipf = [np.minimum(rng.zipf(alpha, draws) - 1, d - 1) for d in dims]
    coords = np.unique(np.stack(zipf, axis=1), axis=0)
    coords = coords[rng.permutation(len(coords))]
    if take is not None:
        coords = coords[:take]
    vals = rng.random(len(coords)) + 0.1
    return rng, coords, vals


@pytest.mark.parametrize("rank", [1, 4, 7, 16, 32, 33])
def test_fused_plain_mttkrp_matches_oracle(monkeypatch, rank):
    """The public 3-mode MTTKRP through the fused fiber kernel (no piece
    sums stored) for every lanes-per-nonzero width (rank 1..32: G = 1, 2, 4,
    8; rank 33 falls back to dview3); a ragged nonzero count leaves a partial
    warp block."""
    dims = (60, 150, 3000)
    rng, coords, vals = _skewed(500 + rank, dims, 80_000, take=45_001)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    for mode in range(3):
        got = K.launch_mttkrp(t, d, mode, "dview")[:, :rank].cpu().numpy()
        assert any(k[0] == "fstream" and k[1] == mode for k in t._cache) == (rank <= 32)
        assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)
    got = alto.mttkrp(t, factors, 1)
    assert_close_rel(got, orc.mttkrp(scoords, svals, factors, 1), rel=1e-12)


@pytest.mark.parametrize("kind", ["fused", "memo0"])
@pytest.mark.parametrize("rank", [1, 5, 16, 32])
def test_memo_producers_match_oracle(monkeypatch, kind, rank):
    """Every producer of the memoised pair (m0, m1) = (1, 2) and (2, 0):
    m0's MTTKRP from its pass and m1's from the stored piece sums equal the
    oracle (pieces cut by segment edges, rows spanning segments, a ragged
    last warp block)."""
    from paper_2403_06348_b200.memo import MemoPlan

    monkeypatch.setenv("ALTO_B200_MEMO_KERNEL", kind)
    dims = (60, 150, 3000)
    rng, coords, vals = _skewed(700 + rank, dims, 200_000, take=70_003)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    factors = [rng.random((n, rank)) for n in dims]
    d = K.DeviceFactors(factors, rank)
    for m0, m1 in ((1, 2), (2, 0)):
        p = MemoPlan(t, rank, m0, m1)
        assert p.kind == kind and p.P < t.nnz
        out0 = torch.zeros((dims[m0], nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
        p.mttkrp_m0(t, d, out0)
        assert_close_rel(out0[:, :rank].cpu().numpy(), orc.mttkrp(scoords, svals, factors, m0), rel=1e-12)
        out1 = torch.zeros((dims[m1], nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
        p.mttkrp_m1(d, out1)
        assert_close_rel(out1[:, :rank].cpu().numpy(), orc.mttkrp(scoords, svals, factors, m1), rel=1e-12)


@pytest.mark.parametrize("rank", [3, 16, 32])
def test_fused_piece_sums_bitwise(monkeypatch, rank):
    """The fused producer writes every piece's T row bit for bit like the
    round-2 memo0 kernel (same per-piece summation order), at the piece's
    consumer slot instead of its T-order row."""
    from paper_2403_06348_b200.memo import MemoPlan

    dims = (50, 70, 4000)
    rng, coords, vals = _skewed(800 + rank, dims, 150_000, take=60_001)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    factors = [rng.random((n, rank)) for n in dims]
    d = K.DeviceFactors(factors, rank)
    monkeypatch.setenv("ALTO_B200_MEMO_KERNEL", "memo0")
    p = MemoPlan(t, rank, 0, 1)
    out = torch.zeros((dims[0], nat.padded_ld(rank)), dtype=torch.float64, device="cuda")
    p.mttkrp_m0(t, d, out)
    ref = p.T[: p.P, :rank].clone()
    pid = p.pid.cpu().numpy().astype(np.int64)
    monkeypatch.setenv("ALTO_B200_MEMO_KERNEL", "fused")
    q = MemoPlan(t, rank, 0, 1)
    assert q.P == p.P
    out2 = torch.zeros_like(out)
    q.mttkrp_m0(t, d, out2)
    g = 1
    while 4 * g < rank:
        g *= 2
    ng = 32 // g
    x = np.arange(q.P)
    seg = x // 512
    slots = (seg // ng) * ng * 512 + ((x % 512) // 4) * 4 * ng + (seg % ng) * 4 + x % 4
    got = q.T[torch.from_numpy(slots).cuda(), :rank]
    assert torch.equal(got, ref[torch.from_numpy(pid).cuda()])
    assert_close_rel(out2[:, :rank].cpu().numpy(), out[:, :rank].cpu().numpy(), rel=1e-13)


def test_fused_producer_single_piece_and_tiny():
    """One nonzero, one row, one fiber: the fused producer's edge cases."""
    from paper_2403_06348_b200.memo import MemoPlan

    rng = np.random.default_rng(5)
    cases = [((3, 4, 5), np.array([[1, 2, 3]])),
             ((4, 30, 40), np.unique(np.stack([np.full(600, 2), rng.integers(0, 30, 600),
                                               rng.integers(0, 40, 600)], 1), axis=0)),
             ((5, 6, 900), np.stack([np.full(700, 3), np.full(700, 4), rng.permutation(900)[:700]], 1))]
    for dims, coords in cases:
        vals = rng.random(len(coords)) + 0.5
        t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
        _keys, svals, scoords = orc.from_coo(dims, coords, vals)
        factors = [rng.random((n, 6)) for n in dims]
        d = K.DeviceFactors(factors, 6)
        p = MemoPlan(t, 6, 0, 1)
        assert p.kind == "fused"
        out0 = torch.zeros((dims[0], nat.padded_ld(6)), dtype=torch.float64, device="cuda")
        p.mttkrp_m0(t, d, out0)
        assert_close_rel(out0[:, :6].cpu().numpy(), orc.mttkrp(scoords, svals, factors, 0), rel=1e-12)
        out1 = torch.zeros((dims[1], nat.padded_ld(6)), dtype=torch.float64, device="cuda")
        p.mttkrp_m1(d, out1)
        assert_close_rel(out1[:, :6].cpu().numpy(), orc.mttkrp(scoords, svals, factors, 1), rel=1e-12)


@pytest.mark.parametrize("fiber", ["long", "short"])
@pytest.mark.parametrize("dims", [(40, 3000, 70, 200), (30, 20, 900, 40, 500)])
@pytest.mark.parametrize("rank", [3, 16, 32, 40])
def test_fused_plain_mttkrp_many_modes(monkeypatch, dims, rank, fiber):
    """4- and 5-mode MTTKRP through the fused fiber kernel (N - 2 gathers per
    nonzero, the shortest other mode's row once per fiber) for every mode;
    rank 40 falls back to dview3. 5 modes are opt-in (measured slower)."""
    monkeypatch.setenv("ALTO_B200_FUSED_MODES", "5")
    monkeypatch.setenv("ALTO_B200_FUSED_FIBER", fiber)
    rng, coords, vals = _skewed(900 + rank + len(dims), dims, 90_000, take=50_003)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    factors = [rng.random((d, rank)) for d in dims]
    d = K.DeviceFactors(factors, rank)
    for mode in range(len(dims)):
        got = K.launch_mttkrp(t, d, mode, "dview")[:, :rank].cpu().numpy()
        fm = K._fused_fiber_mode(t, mode)
        assert (fm != mode) and any(k[0] == "fstream" and k[1] == mode for k in t._cache) == (rank <= 32)
        assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)


def test_fused_plain_mttkrp_many_modes_tiny():
    """One nonzero and one single-fiber row of a 4-mode tensor."""
    assert K._use_fused(alto.AltoTensor.from_coo(alto.CooTensor((3, 4, 5, 6), np.array([[1, 2, 3, 4]]),
                                                                np.ones(1))), 5)
    rng = np.random.default_rng(9)
    cases = [((3, 4, 5, 6), np.array([[1, 2, 3, 4]])),
             ((4, 3, 50, 60), np.stack([np.full(700, 2), np.full(700, 1), rng.integers(0, 50, 700),
                                        rng.integers(0, 60, 700)], 1))]
    for dims, coords in cases:
        coords = np.unique(coords, axis=0)
        vals = rng.random(len(coords)) + 0.5
        t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
        _keys, svals, scoords = orc.from_coo(dims, coords, vals)
        factors = [rng.random((n, 5)) for n in dims]
        d = K.DeviceFactors(factors, 5)
        for mode in range(4):
            got = K.launch_mttkrp(t, d, mode, "dview")[:, :5].cpu().numpy()
            assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)


@pytest.mark.parametrize("dims,rank", [((60, 150, 3000), 16), ((7, 5000, 3), 4), ((40, 30, 20, 900), 32),
                                       ((9, 8, 7, 6, 500), 8), ((1, 1, 70_000), 2),
                                       ((2_000_000, 1_500_000, 3_000_000, 168), 32)])
def test_fused_stream_build_equals_three_pass_build(monkeypatch, dims, rank):
    """The one-call stream build (sort + gather / decode / interleave in one
    pass, alto_fused_stream_build) writes bit for bit what the permuted copy
    + decoded view + interleave passes write, for 3-5 modes, 64- and 128-bit
    keys, every lanes-per-nonzero width and a ragged last warp block (the
    order is the reference's stable sort, pkg/src/alto/partition.py:185-188)."""
    from paper_2403_06348_b200 import partition as P

    rng, coords, vals = _skewed(77, dims, 60_000, alpha=1.2, take=33_333)
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    for mode in range(len(dims)):
        for fm in {K._fused_fiber_mode(t, mode), (mode + 1) % len(dims)}:
            monkeypatch.setenv("ALTO_B200_STREAM_BUILD", "legacy")
            t._cache.clear()
            old = [x.clone() for x in P.device_fused_stream(t, mode, fm, rank)]
            monkeypatch.setenv("ALTO_B200_STREAM_BUILD", "fused")
            t._cache.clear()
            new = P.device_fused_stream(t, mode, fm, rank)
            for a, b in zip(old, new):
                assert a.shape == b.shape
                assert torch.equal(a.view(torch.uint8), b.contiguous().view(torch.uint8))


@pytest.mark.parametrize("nnz", [1, 2, 3, 5, 511, 512, 513])
def test_fused_stream_build_tiny_tensors(monkeypatch, nnz):
    """Fewer nonzeros than one quad / exactly one segment / one past it: the
    one-pass build equals the three-pass build and the MTTKRP the oracle."""
    from paper_2403_06348_b200 import partition as P

    dims = (6, 5, 40)
    rng = np.random.default_rng(nnz)
    flat = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    coords = np.stack(np.unravel_index(flat, dims), axis=1).astype(np.int64)
    vals = rng.random(nnz) + 0.5
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    rank = 5
    factors = [rng.random((d, rank)) for d in dims]
    for mode in range(3):
        fm = K._fused_fiber_mode(t, mode)
        monkeypatch.setenv("ALTO_B200_STREAM_BUILD", "legacy")
        t._cache.clear()
        old = [x.clone() for x in P.device_fused_stream(t, mode, fm, rank)]
        monkeypatch.setenv("ALTO_B200_STREAM_BUILD", "fused")
        t._cache.clear()
        new = P.device_fused_stream(t, mode, fm, rank)
        for a, b in zip(old, new):
            assert torch.equal(a.view(torch.uint8), b.contiguous().view(torch.uint8))
        got = alto.mttkrp(t, factors, mode)
        assert_close_rel(got, orc.mttkrp(scoords, svals, factors, mode), rel=1e-12)
