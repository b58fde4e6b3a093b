"""World-size-2 sharding of the ALTO stream on CPU (gloo backend).

Each rank takes its balanced ALTO-ordered slice (distributed.shard_range),
computes a partial MTTKRP / Phi with the oracle standing in for the device
kernel, and the partials are summed with distributed.allreduce_; the result
must equal the single-process computation. Also covers the replicated CP-ALS
step that follows the all-reduce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import random_sparse
from oracle import alto_oracle as orc
from paper_2403_06348_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    rng = np.random.default_rng(42)
    dims = (23, 17, 31)
    coords, vals = random_sparse(rng, dims, 900, kind="positive")
    cc, cv = orc.canonicalize(coords, vals)
    keys, svals, scoords = orc.from_coo(dims, cc, cv)
    factors = [rng.random((d, 6)) for d in dims]
    return dims, scoords, svals, factors


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, coords, vals, factors = _problem()
        a, b = D.shard_range(len(vals), world, rank)
        res = {}
        for mode in range(3):
            part = orc.mttkrp(coords[a:b], vals[a:b], factors, mode)
            t = torch.from_numpy(part.copy())
            D.allreduce_(t)
            res[f"m{mode}"] = t.numpy()
            scaled = np.full((dims[mode], 6), 0.5)
            ppart = orc.phi(coords[a:b], vals[a:b], scaled, factors, mode)
            tp = torch.from_numpy(ppart.copy())
            D.allreduce_(tp)
            res[f"phi{mode}"] = tp.numpy()
        res["kmax"] = np.asarray(D.allreduce_max(float(rank) + 0.5))
        if rank == 0:
            np.savez(out_path, **res)
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_stream():
    for M in (1, 7, 1000, 76_000_000):
        for world in (1, 2, 4, 8):
            if world > M:
                continue
            spans = [D.shard_range(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_allreduce_matches_single_process(tmp_path):
    out = tmp_path / "r0.npz"
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(out)), nprocs=2, join=True)
    got = np.load(out)
    dims, coords, vals, factors = _problem()
    for mode in range(3):
        want = orc.mttkrp(coords, vals, factors, mode)
        np.testing.assert_allclose(got[f"m{mode}"], want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
        scaled = np.full((dims[mode], 6), 0.5)
        pwant = orc.phi(coords, vals, scaled, factors, mode)
        np.testing.assert_allclose(got[f"phi{mode}"], pwant, rtol=1e-12, atol=1e-12 * np.abs(pwant).max())
    assert float(got["kmax"]) == 1.5


def test_rank_shards_are_line_segments():
    dims, coords, vals, factors = _problem()
    bounds, lo, hi, _ = orc.segments(coords, 2)
    for r in range(2):
        a, b = D.shard_range(len(vals), 2, r)
        assert (a, b) == (bounds[r], bounds[r + 1])
        assert np.array_equal(coords[a:b].min(axis=0), lo[r])
        assert np.array_equal(coords[a:b].max(axis=0), hi[r])


def _rows_worker(rank, world, port, out_path):
    """Row-owner CP-ALS (distributed.RowComm): partial MTTKRP per shard,
    reduce-scatter to row owners (matrices padded to world * chunk rows),
    owner-side solve of its rows, all-reduce of the raw Gram (column norms =
    sqrt of its diagonal), normalisation, all-gather. The oracle's kernels
    and numpy's Cholesky stand in for the device kernels."""
    import scipy.linalg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, coords, vals, _ = _problem()
        R = 6
        a, b = D.shard_range(len(vals), world, rank)
        rc = D.RowComm()
        w, factors = orc.normalized(*orc.init_factors(dims, R, 3), ord=2)
        grams = [f.T @ f for f in factors]
        for _sweep in range(2):
            for n in range(3):
                v = orc._hadamard(grams, skip=n)
                part = orc.mttkrp(coords[a:b], vals[a:b], factors, n)
                full = torch.zeros((rc.padded(dims[n]), R), dtype=torch.float64)
                full[: dims[n]] = torch.from_numpy(part)
                blk = torch.empty((rc.chunk(dims[n]), R), dtype=torch.float64)
                rc.reduce_scatter(blk, full)
                ab = scipy.linalg.cho_solve(scipy.linalg.cho_factor(v), blk.numpy().T).T
                raw = torch.from_numpy(ab.T @ ab)
                rc.all_reduce(raw)
                norms = np.sqrt(np.diag(raw.numpy()))
                safe = np.where(norms == 0.0, 1.0, norms)
                ab = ab / safe
                gathered = torch.zeros_like(full)
                rc.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(ab)))
                factors[n] = gathered.numpy()[: dims[n]].copy()
                grams[n] = raw.numpy() / np.outer(safe, safe)
                w = norms
        if rank == 0:
            np.savez(out_path, w=w, **{f"f{n}": f for n, f in enumerate(factors)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_owner_update_matches_single_process(tmp_path, world):
    out = tmp_path / "rows.npz"
    mp.spawn(_rows_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    dims, coords, vals, _ = _problem()
    w, fs, _fits = orc.cp_als(dims, coords, vals, 6, 2, seed=3)
    np.testing.assert_allclose(got["w"], w, rtol=1e-9)
    for n in range(3):
        np.testing.assert_allclose(got[f"f{n}"], fs[n], rtol=0, atol=1e-9 * np.abs(fs[n]).max())


def _timeout_worker(rank, world, port, out_path):
    import datetime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=3))
    msg = "no error"
    try:
        if rank == 0:  # rank 1 never joins this collective
            try:
                D.allreduce_(torch.ones(4, dtype=torch.float64))
            except RuntimeError as e:
                msg = f"{type(e).__name__}: {e}"
            with open(out_path, "w") as f:
                f.write(msg)
        else:
            import time

            time.sleep(6)
    finally:
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def test_collective_timeout_maps_to_runtime_error(tmp_path):
    """A collective a peer never joins times out and surfaces as the
    reference's RuntimeError for CUDA / NCCL failures, naming the collective."""
    out = tmp_path / "msg.txt"
    mp.spawn(_timeout_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    msg = out.read_text()
    assert msg.startswith("RuntimeError: all_reduce failed across ranks"), msg
