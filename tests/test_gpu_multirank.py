"""The multi-rank drivers on real kernels: two ranks share the one GPU of the
test box with the gloo backend (collectives staged through the host; NCCL is
the production backend and cannot put two ranks on one device). Each rank
takes its balanced ALTO-ordered shard, runs the GPU MTTKRP / Phi on it and
sums the partials; CP-ALS and CP-APR must then match the single-process run
(same kernels, different summation split: 1e-9 relative)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import assert_close_rel, random_sparse

pytestmark = pytest.mark.gpu

DIMS = (60, 45, 70)
KINDS = ("als", "als_rows", "apr", "apr_tau")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tensors(kind):
    import paper_2403_06348_b200 as alto

    als = kind.startswith("als")
    rng = np.random.default_rng(11 if als else 12)
    coords, vals = random_sparse(rng, DIMS, 6000, kind="positive" if als else "counts")
    return alto.AltoTensor.from_coo(alto.CooTensor(DIMS, coords, vals))


def _run(kind, world=1, rank=0):
    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import distributed as D
    from paper_2403_06348_b200.cpd import als as ALS
    from paper_2403_06348_b200.cpd import apr as APR

    full = _tensors(kind)
    t = D.shard_tensor(full, world, rank) if world > 1 else full
    reduce = D.allreduce_ if world > 1 else None
    if kind in ("als", "als_rows"):
        norm = float(full._vals @ full._vals)
        if kind == "als_rows":  # reduce-scatter to row owners, owner solve, all-gather
            comm = {"row_comm": D.RowComm()} if world > 1 else {}
        else:
            comm = {"reduce": reduce}
        st = ALS.AlsState(t, alto.CpAlsConfig(rank=5, max_iters=6, seed=3), norm_x_sq=norm, memo=True, **comm)
        fits = []
        for _ in range(6):
            st.sweep()
            fits.append(st.fit()[0])
        m = st.model()
        return {"fits": np.asarray(fits), "weights": m.weights, **{f"f{n}": f for n, f in enumerate(m.factors)}}
    # "apr_tau": a loose tau, so inner loops break early (at it = 0 and it > 0)
    # and the next outer's shift reads the Phi of the converged iteration
    tau = 0.2 if kind == "apr_tau" else 1e-4
    st = APR.AprState(t, alto.CpAprConfig(rank=4, max_outer=4, max_inner=10, seed=3, tau=tau), reduce=reduce)
    for _ in range(4):
        st.outer()
    m = st.model()
    return {"loglik": np.asarray(st.loglik_trace), "inner": np.asarray(st.inner_counts),
            "weights": m.weights, **{f"f{n}": f for n, f in enumerate(m.factors)}}


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for kind in KINDS:
            res = _run(kind, world, rank)
            if rank == 0:
                np.savez(f"{out}_{kind}.npz", **res)
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_process(tmp_path):
    out = str(tmp_path / "r0")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for kind in KINDS:
        got = np.load(f"{out}_{kind}.npz")
        want = _run(kind)
        if kind == "apr_tau":
            assert (want["inner"] < 10).any()  # some inner loop broke early
        for key, w in want.items():
            if key == "inner":
                assert np.array_equal(got[key], w)
            else:
                assert_close_rel(got[key], w, rel=1e-9)


def _construct_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_06348_b200 import distributed as D

        for tag, dims in (("w64", (300, 70, 4000)), ("w128", (2**22, 2**21, 2**22))):
            coords, vals = _construct_problem(dims)
            mine = np.arange(len(vals)) % world == rank  # an arbitrary (unsorted) slice per rank
            shard, (a, b) = D.build_sharded(dims, coords[mine], vals[mine])
            np.savez(f"{out}_{tag}_{rank}.npz", keys=shard._keys.cpu().numpy(), vals=shard._vals.cpu().numpy(),
                     a=a, b=b)
    finally:
        dist.destroy_process_group()


def _construct_problem(dims):
    rng = np.random.default_rng(sum(dims) % 1000)
    coords, vals = random_sparse(rng, dims, 20_011, kind="positive")
    _u, first = np.unique(coords, axis=0, return_index=True)  # canonical: unique coordinates
    keep = np.sort(first)
    return coords[keep], vals[keep]


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_construction_cuts_single_gpu_shards(tmp_path, world):
    """build_sharded: each rank ends with exactly the ALTO-ordered range
    [b_r, b_{r+1}) of balanced_bounds(M, world) of the single-GPU build,
    for 64- and 128-bit keys."""
    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200.partition import balanced_bounds

    out = str(tmp_path / "c")
    mp.spawn(_construct_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for tag, dims in (("w64", (300, 70, 4000)), ("w128", (2**22, 2**21, 2**22))):
        coords, vals = _construct_problem(dims)
        full = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
        keys, fvals = full._keys.cpu().numpy(), full._vals.cpu().numpy()
        bounds = balanced_bounds(full.nnz, world)
        for r in range(world):
            got = np.load(f"{out}_{tag}_{r}.npz")
            assert (int(got["a"]), int(got["b"])) == (bounds[r], bounds[r + 1])
            assert np.array_equal(got["keys"], keys[bounds[r]:bounds[r + 1]])
            assert np.array_equal(got["vals"], fvals[bounds[r]:bounds[r + 1]])
