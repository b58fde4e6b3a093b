"""NCCL through the C ABI (alto_nccl_*, alto_mttkrp_sharded; SURVEY.md 8(b),
8(e)). The test box has one GPU and NCCL cannot put two ranks on one
device, so the communicator here has one rank: the collectives are then
identities and the sharded MTTKRP must equal the oracle's MTTKRP of the
whole tensor. The sharding arithmetic itself (shards of balanced_bounds,
row-owner blocks, several ranks) is covered by test_gpu_multirank.py and
test_multirank_gloo.py."""

import numpy as np
import pytest
import torch

import paper_2403_06348_b200 as alto
from conftest import assert_close_rel, random_sparse
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import distributed as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = D.NativeComm()
    yield c
    c.close()


def _case(dims, nnz, rank, seed):
    rng = np.random.default_rng(seed)
    coords, vals = random_sparse(rng, dims, nnz, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    facs = [rng.random((d, rank)) for d in dims]
    ocoords, ovals = orc.canonicalize(coords, vals)
    _, svals, scoords = orc.from_coo(dims, ocoords, ovals)
    return t, facs, scoords, svals


def test_one_rank_communicator(comm):
    assert (comm.world, comm.rank) == (1, 0)
    comm.check()
    x = torch.arange(1000, dtype=torch.float64, device="cuda")
    assert torch.equal(comm.all_reduce(x.clone()), x)
    full = torch.rand(64, 8, dtype=torch.float64, device="cuda")
    blk = torch.empty_like(full)
    comm.reduce_scatter(blk, full)
    assert torch.equal(blk, full)
    out = torch.empty_like(full)
    comm.all_gather(out, blk)
    assert torch.equal(out, full)
    flags = torch.tensor([0, 3, 0, 1], dtype=torch.int32, device="cuda")
    assert comm.all_reduce_max(flags).tolist() == [0, 1, 0, 1]


def test_collective_argument_errors(comm):
    with pytest.raises(ValueError):
        comm.all_reduce(torch.zeros(4, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        comm.reduce_scatter(torch.zeros(3, dtype=torch.float64, device="cuda"),
                            torch.zeros(4, dtype=torch.float64, device="cuda"))


def test_all_reduce_in_a_cuda_graph(comm):
    x = torch.ones(4096, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        comm.all_reduce(x)  # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        x.mul_(2.0)
        comm.all_reduce(x)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, torch.full_like(x, 8.0))


@pytest.mark.parametrize("kernel", ["segment", "atomic"])
@pytest.mark.parametrize("owner_rows", [False, True])
@pytest.mark.parametrize("dims,rank", [((37, 23, 41), 16), ((12, 9, 7, 5), 5), ((30, 2, 17), 33)])
def test_mttkrp_sharded_matches_oracle(comm, kernel, owner_rows, dims, rank):
    t, facs, scoords, svals = _case(dims, 2500, rank, seed=len(dims) * 100 + rank)
    for mode in range(len(dims)):
        got = D.mttkrp_sharded(t, facs, mode, comm, kernel=kernel, owner_rows=owner_rows)
        got = got[: dims[mode], :rank].cpu().numpy()
        want = orc.mttkrp(scoords, svals, facs, mode, "sequential")
        assert_close_rel(got, want, 1e-12)


def test_mttkrp_sharded_empty_shard(comm):
    # more ranks than nonzeros: some ALTO-ordered shards are empty
    full = alto.AltoTensor.from_coo(alto.CooTensor((5, 4, 3), [[0, 1, 2], [4, 3, 0]], [1.0, 2.0]))
    empty = [r for r in range(8) if D.shard_range(full.nnz, 8, r)[0] == D.shard_range(full.nnz, 8, r)[1]]
    t = D.shard_tensor(full, 8, empty[0])
    assert t.nnz == 0
    facs = [np.ones((d, 4)) for d in (5, 4, 3)]
    out = D.mttkrp_sharded(t, facs, 1, comm, kernel="segment")
    assert out.shape[0] == 4 and float(out.abs().sum()) == 0.0


def test_mttkrp_sharded_rejects_bad_input(comm):
    t, facs, _, _ = _case((10, 11, 12), 300, 4, seed=5)
    with pytest.raises(ValueError, match="mode 3 out of range"):
        D.mttkrp_sharded(t, facs, 3, comm)
    with pytest.raises(ValueError):
        D.mttkrp_sharded(t, facs, 0, comm, kernel="dense")
    bad = [f.copy() for f in facs]
    bad[2][0, 0] = np.nan
    with pytest.raises(ValueError):
        D.mttkrp_sharded(t, bad, 0, comm)
        torch.cuda.synchronize()


def test_cp_als_row_owners_over_native_comm(comm):
    from paper_2403_06348_b200.cpd import als as ALS

    t, _, _, _ = _case((60, 45, 70), 6000, 5, seed=9)
    norm = float(t._vals @ t._vals)
    cfg = alto.CpAlsConfig(rank=5, max_iters=5, seed=3)
    ref = ALS.AlsState(t, cfg, norm_x_sq=norm, memo=True)
    nat_ = ALS.AlsState(t, cfg, norm_x_sq=norm, memo=True, row_comm=comm)
    for _ in range(5):
        ref.sweep()
        nat_.sweep()
    assert_close_rel(nat_.fit()[0], ref.fit()[0], 1e-12, scale=1.0)
    m1, m2 = nat_.model(), ref.model()
    assert_close_rel(m1.weights, m2.weights, 1e-9)
    for a, b in zip(m1.factors, m2.factors):
        assert_close_rel(a, b, 1e-9)


def test_cp_als_allreduce_over_native_comm_in_graphs(comm):
    from paper_2403_06348_b200.cpd import als as ALS

    t, _, _, _ = _case((60, 45, 70), 6000, 5, seed=10)
    norm = float(t._vals @ t._vals)
    cfg = alto.CpAlsConfig(rank=5, max_iters=5, seed=4)
    ref = ALS.AlsState(t, cfg, norm_x_sq=norm, memo=True)
    nat_ = ALS.AlsState(t, cfg, norm_x_sq=norm, memo=True, reduce=comm.all_reduce)
    assert nat_._graph_capturable()
    for _ in range(5):
        ref.sweep()
        nat_.sweep()
    assert_close_rel(nat_.fit()[0], ref.fit()[0], 1e-12, scale=1.0)
    for a, b in zip(nat_.model().factors, ref.model().factors):
        assert_close_rel(a, b, 1e-9)


@pytest.mark.parametrize("tau", [1e-4, 0.2])
def test_cp_apr_over_native_comm_in_graphs(comm, tau):
    """The multi-rank device inner loop (all-reduce of every Phi partial,
    conditional keep of the last reduced Phi) captured in the outer-iteration
    graph; tau 0.2 breaks inner loops early."""
    from paper_2403_06348_b200.cpd import apr as APR

    rng = np.random.default_rng(12)
    dims = (60, 45, 70)
    coords, vals = random_sparse(rng, dims, 6000, kind="counts")
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
    cfg = alto.CpAprConfig(rank=4, max_outer=5, max_inner=10, seed=3, tau=tau)
    ref = APR.AprState(t, cfg)
    nat_ = APR.AprState(t, cfg, reduce=comm.all_reduce)
    assert nat_._graph_ok()
    for _ in range(5):
        ref.outer()
        nat_.outer()
    assert nat_._graph is not None
    assert nat_.inner_counts == ref.inner_counts
    assert_close_rel(nat_.loglik_trace, ref.loglik_trace, 1e-12)
    for a, b in zip(nat_.model().factors, ref.model().factors):
        assert_close_rel(a, b, 1e-9)
