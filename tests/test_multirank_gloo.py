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
