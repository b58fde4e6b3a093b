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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tensors(kind):
    import paper_2403_06348_b200 as alto

    rng = np.random.default_rng(11 if kind == "als" else 12)
    coords, vals = random_sparse(rng, DIMS, 6000, kind="positive" if kind == "als" else "counts")
    return alto.AltoTensor.from_coo(alto.CooTensor(DIMS, coords, vals))


def _run(kind, world=1, rank=0):
    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import distributed as D
    from paper_2403_06348_b200.cpd import als as ALS
    from paper_2403_06348_b200.cpd import apr as APR

    full = _tensors(kind)
    t = D.shard_tensor(full, world, rank) if world > 1 else full
    reduce = D.allreduce_ if world > 1 else None
    if kind == "als":
        norm = float(full._vals @ full._vals)
        st = ALS.AlsState(t, alto.CpAlsConfig(rank=5, max_iters=6, seed=3), reduce=reduce, norm_x_sq=norm)
        fits = []
        for _ in range(6):
            st.sweep()
            fits.append(st.fit()[0])
        m = st.model()
        return {"fits": np.asarray(fits), "weights": m.weights, **{f"f{n}": f for n, f in enumerate(m.factors)}}
    st = APR.AprState(t, alto.CpAprConfig(rank=4, max_outer=4, max_inner=10, seed=3), reduce=reduce)
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
        for kind in ("als", "apr"):
            res = _run(kind, world, rank)
            if rank == 0:
                np.savez(f"{out}_{kind}.npz", **res)
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_process(tmp_path):
    out = str(tmp_path / "r0")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for kind in ("als", "apr"):
        got = np.load(f"{out}_{kind}.npz")
        want = _run(kind)
        for key, w in want.items():
            if key == "inner":
                assert np.array_equal(got[key], w)
            else:
                assert_close_rel(got[key], w, rel=1e-9)
