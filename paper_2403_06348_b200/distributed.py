"""Multi-GPU sharding of the ALTO nonzero stream.

One process per GPU. Rank r owns the contiguous ALTO-ordered slice
[bounds[r], bounds[r+1]) with bounds = balanced_bounds(M, world) -- a line
segment at L = world (pkg/src/alto/partition.py:69-75). Every rank computes
a factor-sized partial MTTKRP / Phi over its slice; the partials are summed
with one NCCL all-reduce over NVLink (reduce-scatter + all-gather of the
updated rows collapsed into one collective, since the R x R solve is
replicated), after which every rank holds identical factors.

The same code runs on CPU tensors with the gloo backend (tests).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .partition import balanced_bounds


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    b = balanced_bounds(M, world)
    return int(b[rank]), int(b[rank + 1])


def shard_tensor(alto, world: int, rank: int):
    """This rank's slice of a device AltoTensor (views, no copy)."""
    from .tensor import AltoTensor

    a, b = shard_range(alto.nnz, world, rank)
    return AltoTensor(alto.layout, alto._keys[a:b], alto._vals[a:b], _validate=False)


def _failed(what: str, err: Exception) -> RuntimeError:
    """NCCL / gloo failures (timeouts, aborts, a dead peer) surface as the
    reference's RuntimeError for CUDA/NCCL errors."""
    return RuntimeError(f"{what} failed across ranks: {type(err).__name__}: {err}")


def _collective(t, op, group):
    """all_reduce in place; NCCL reduces device tensors directly, gloo (tests,
    including several ranks sharing one GPU) stages them through the host."""
    import torch.distributed as dist

    try:
        if dist.get_backend(group) == "gloo" and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=group)
    except RuntimeError as e:
        raise _failed("all_reduce", e) from e
    return t


class RowComm:
    """Row-owner collectives of the sharded CP-ALS update:
    the factor-sized MTTKRP partials are reduce-scattered so that rank r
    owns rows [r c, (r + 1) c) of mode n (c = ceil(I_n / W), matrices padded
    to W c rows), the owner solves its rows (the solve is row-separable),
    the R x R raw Gram is all-reduced (column norms = sqrt of its diagonal)
    and the normalised blocks are all-gathered. Per mode and rank this moves
    the same bytes as one all-reduce of the partial (reduce-scatter +
    all-gather), but the solve, Gram and scaling run on 1/W of the rows.
    NCCL for device tensors; gloo stages through the host (tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.gloo = dist.get_backend(group) == "gloo"

    def chunk(self, rows: int) -> int:
        return -(-int(rows) // self.world)

    def padded(self, rows: int) -> int:
        return self.chunk(rows) * self.world

    def block(self, full):
        """This rank's row block (a view) of a padded matrix."""
        c = full.shape[0] // self.world
        return full[self.rank * c:(self.rank + 1) * c]

    def reduce_scatter(self, blk, full):
        import torch.distributed as dist

        try:
            if self.gloo and full.is_cuda:
                h = blk.new_empty(blk.shape, device="cpu")
                dist.reduce_scatter_tensor(h, full.cpu(), group=self.group)
                blk.copy_(h)
            else:
                dist.reduce_scatter_tensor(blk, full, group=self.group)
        except RuntimeError as e:
            raise _failed("reduce_scatter", e) from e
        return blk

    def all_gather(self, full, blk):
        import torch.distributed as dist

        try:
            if self.gloo and full.is_cuda:
                h = full.new_empty(full.shape, device="cpu")
                dist.all_gather_into_tensor(h, blk.cpu(), group=self.group)
                full.copy_(h)
            else:
                dist.all_gather_into_tensor(full, blk, group=self.group)
        except RuntimeError as e:
            raise _failed("all_gather", e) from e
        return full

    def all_reduce(self, t):
        import torch.distributed as dist

        return _collective(t, dist.ReduceOp.SUM, self.group)

    def all_reduce_max(self, t):
        import torch.distributed as dist

        return _collective(t, dist.ReduceOp.MAX, self.group)


def _active(group) -> bool:
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def allreduce_(t, group=None):
    """In-place sum over ranks (NCCL over NVLink for CUDA tensors)."""
    import torch.distributed as dist

    if _active(group):
        _collective(t, dist.ReduceOp.SUM, group)
    return t


def allreduce_max(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not _active(group):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    _collective(t, dist.ReduceOp.MAX, group)
    return float(t.item())


def agree_kernels(kernels: list, group=None) -> list:
    """Make every rank use the same per-mode kernel. Each rank picks its
    kernel from its own free memory and cache (``select_gpu_kernel``), and
    the CP-APR inner loop issues a different number of collectives per
    kernel (device-driven vs host-driven), so a disagreement near the
    memory threshold would hang NCCL: modes where the ranks differ fall
    back to the view-free ``atomic`` kernel everywhere."""
    import torch

    from .kernels import GPU_KERNELS

    if not _active(group):
        return list(kernels)
    names = list(GPU_KERNELS) + ["exact-seq", "exact-rec", "exact-output"]
    codes = [names.index(k) for k in kernels]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    hi = torch.tensor(codes, dtype=torch.int64, device=dev)
    lo = -hi.clone()
    import torch.distributed as dist

    _collective(hi, dist.ReduceOp.MAX, group)
    _collective(lo, dist.ReduceOp.MAX, group)
    return [k if int(a) == -int(b) else "atomic" for k, a, b in zip(kernels, hi.tolist(), lo.tolist())]


def reduce_partials_numpy(parts: list[np.ndarray]) -> np.ndarray:
    """Fixed-order host sum of per-rank partials (reference for tests)."""
    out = np.zeros_like(parts[0])
    for p in parts:
        out += p
    return out


# ---------------------------------------------------------------------------
# distributed construction: every rank holds an arbitrary
# slice of a canonical COO; afterwards rank r holds exactly the ALTO-ordered
# range [b_r, b_{r+1}) of balanced_bounds(M, world) -- the same shard the
# single-GPU build would cut.


def _alltoall(out, inp, out_splits, in_splits, group):
    import torch.distributed as dist

    try:
        if dist.get_backend(group) == "gloo" and inp.is_cuda:
            h_out = out.new_empty(out.shape, device="cpu")
            dist.all_to_all_single(h_out, inp.cpu(), out_splits, in_splits, group=group)
            out.copy_(h_out)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    except RuntimeError as e:
        raise _failed("all_to_all", e) from e
    return out


def _int_to_words(q: int, words: int) -> list:
    mask = (1 << 64) - 1
    w = [q & mask, (q >> 64) & mask][:words]
    return [x - (1 << 64) if x >= 1 << 63 else x for x in w]  # int64 bit patterns


def _count_less(keys, words: int, queries: list):
    """Per query key (Python int): how many of the ascending keys are below it."""
    import ctypes

    import torch

    t = torch
    n = keys.shape[0]
    top = 1 << (64 * words)
    # a query past the key space counts every key (x + 1 can reach 2^(64 w))
    clipped = [min(k, top - 1) for k in queries]
    q = t.tensor([w for k in clipped for w in _int_to_words(k, words)], dtype=t.int64, device=keys.device)
    out = t.empty(len(queries), dtype=t.int64, device=keys.device)
    nat.call("alto_count_less", 64 * words, nat.ptr(keys), n, nat.ptr(q), len(queries), nat.ptr(out),
             nat.stream_ptr())
    over = [i for i, k in enumerate(queries) if k >= top]
    if over:
        out[over] = n
    return out


def build_sharded(shape, coords, values, group=None):
    """Distributed ALTO construction: encode + sort this rank's slice, find
    the global splitter keys (the keys at positions balanced_bounds(M, W)[1:-1])
    by a bisection over the key space with one all-reduce of W-1 counts per
    key bit, exchange the ranges with one all-to-all, sort what arrived.
    Coordinates must be canonical (unique) across ranks. Returns
    (AltoTensor shard, (first, stop) global positions)."""
    import torch
    import torch.distributed as dist

    from .encoding import as_shape, build_layout
    from .tensor import AltoTensor, _to_device, device_encode, sort_pairs

    t = torch
    shape = as_shape(shape)
    layout = build_layout(shape)
    words = layout.word_bits // 64
    W = dist.get_world_size(group)
    r = dist.get_rank(group)
    dc = _to_device(coords, t.int64).reshape(-1, shape.ndim)
    keys = device_encode(layout, dc)
    vals = _to_device(values, t.float64).clone()
    sort_pairs(layout, keys, vals)
    m = t.tensor([vals.shape[0]], dtype=t.int64, device=vals.device)
    allreduce_(m, group)
    M = int(m.item())
    bounds = balanced_bounds(M, W)
    targets = [int(b) for b in bounds[1:-1]]
    # bisection: smallest key k with count(keys < k + 1) > target (unique keys)
    lo = [0] * len(targets)
    hi = [(1 << layout.total_bits) - 1] * len(targets)
    while any(a < b for a, b in zip(lo, hi)):
        mids = [(a + b) // 2 for a, b in zip(lo, hi)]
        c = _count_less(keys, words, [x + 1 for x in mids])
        allreduce_(c, group)
        cl = c.tolist()
        for i, (cnt, mid) in enumerate(zip(cl, mids)):
            if lo[i] >= hi[i]:
                continue
            if cnt > targets[i]:
                hi[i] = mid
            else:
                lo[i] = mid + 1
    splitters = lo
    pos = _count_less(keys, words, splitters).tolist() if splitters else []
    edges = [0] + pos + [vals.shape[0]]
    send = [edges[i + 1] - edges[i] for i in range(W)]
    send_t = t.tensor(send, dtype=t.int64, device=vals.device)
    recv_t = t.empty_like(send_t)
    _alltoall(recv_t, send_t, [1] * W, [1] * W, group)
    recv = recv_t.tolist()
    n = sum(recv)
    kout = t.empty((n, 2) if words == 2 else (n,), dtype=t.int64, device=keys.device)
    vout = t.empty(n, dtype=t.float64, device=vals.device)
    _alltoall(kout, keys, recv, send, group)
    _alltoall(vout, vals, recv, send, group)
    sort_pairs(layout, kout, vout)
    return AltoTensor(layout, kout, vout, _validate=False), (int(bounds[r]), int(bounds[r + 1]))


# ---------------------------------------------------------------------------
# NCCL through the C ABI (include/alto_b200.h alto_nccl_*, csrc/comm.cu):
# the communicator belongs to the library, so the sharded MTTKRP entry
# (alto_mttkrp_sharded) and the CP-ALS row-owner collectives
# run without torch.distributed's process-group machinery on the data path;
# torch.distributed only ships the unique id once.


class NativeComm:
    """An NCCL communicator created by ``alto_nccl_comm_init`` over the ranks
    of ``group`` (or a standalone one-rank communicator when no process
    group is initialised). Collectives take fp64 CUDA tensors and run on the
    current stream (capturable in CUDA graphs); failures raise RuntimeError.
    Same collective methods as ``RowComm`` (sum only)."""

    UNIQUE_ID_BYTES = 128

    def __init__(self, group=None):
        import ctypes

        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        uid = (ctypes.c_uint8 * self.UNIQUE_ID_BYTES)()
        if self.rank == 0:
            nat.call("alto_nccl_unique_id", ctypes.cast(uid, ctypes.c_void_p), self.UNIQUE_ID_BYTES)
        if self.world > 1:
            box = [bytes(uid)]
            try:
                dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                           group=group)
            except RuntimeError as e:
                raise _failed("unique-id broadcast", e) from e
            ctypes.memmove(uid, box[0], self.UNIQUE_ID_BYTES)
        comm = ctypes.c_void_p(0)
        nat.call("alto_nccl_comm_init", ctypes.cast(uid, ctypes.c_void_p), self.UNIQUE_ID_BYTES, self.world,
                 self.rank, ctypes.byref(comm))
        self.comm = comm.value
        self.gloo = False

    # RowComm's row-block helpers
    def chunk(self, rows: int) -> int:
        return -(-int(rows) // self.world)

    def padded(self, rows: int) -> int:
        return self.chunk(rows) * self.world

    def block(self, full):
        c = full.shape[0] // self.world
        return full[self.rank * c:(self.rank + 1) * c]

    @staticmethod
    def _f64(t, what):
        if not (t.is_cuda and t.dtype == nat.torch().float64 and t.is_contiguous()):
            raise ValueError(f"{what}: NativeComm collectives take contiguous fp64 CUDA tensors")

    def all_reduce(self, t):
        self._f64(t, "all_reduce")
        nat.call("alto_nccl_allreduce_f64", nat.ptr(t), t.numel(), self.comm, nat.stream_ptr())
        return t

    def reduce_scatter(self, blk, full):
        self._f64(blk, "reduce_scatter")
        self._f64(full, "reduce_scatter")
        if full.numel() != blk.numel() * self.world:
            raise ValueError("reduce_scatter: full must hold world x block elements")
        nat.call("alto_nccl_reduce_scatter_f64", nat.ptr(full), nat.ptr(blk), blk.numel(), self.comm,
                 nat.stream_ptr())
        return blk

    def all_gather(self, full, blk):
        self._f64(blk, "all_gather")
        self._f64(full, "all_gather")
        if full.numel() != blk.numel() * self.world:
            raise ValueError("all_gather: full must hold world x block elements")
        nat.call("alto_nccl_allgather_f64", nat.ptr(blk), nat.ptr(full), blk.numel(), self.comm,
                 nat.stream_ptr())
        return full

    def all_reduce_max(self, t):
        # flags only (RowComm contract): max of 0/1 int32 flags = OR, via a
        # fp64 sum (exact for counts < 2^53)
        f = t.to(nat.torch().float64)
        self.all_reduce(f)
        t.copy_((f > 0).to(t.dtype))
        return t

    def check(self) -> None:
        """Raise RuntimeError when the communicator saw an asynchronous error."""
        nat.call("alto_nccl_check", self.comm)

    def close(self, abort: bool = False) -> None:
        if getattr(self, "comm", None):
            nat.call("alto_nccl_comm_destroy", self.comm, int(abort))
            self.comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mttkrp_sharded(shard, factors, mode: int, comm: "NativeComm", *, kernel: str = "segment",
                   owner_rows: bool = False):
    """``alto_mttkrp_sharded`` on this rank's ALTO-ordered shard: the partial
    MTTKRP summed over ``comm``'s ranks (``owner_rows``: reduce-scattered to
    the row owners, rank r's rows [r c, (r + 1) c) valid). ``kernel``:
    'segment' (the ALTO line-segment kernel, privatised when the widest
    interval fits in shared memory) or 'atomic' (key stream, fp64
    reductions). Returns the device output (rows, padded to world * c rows
    with ``owner_rows``)."""
    import ctypes

    from .kernels import DeviceFactors, _prepare, segment_plan
    from .validation import check_mode

    t = nat.torch()
    check_mode(mode, shard.ndim)
    if isinstance(factors, DeviceFactors):
        dfac = factors
    else:
        factors, rank = _prepare(shard, factors, mode)
        dfac = DeviceFactors(factors, rank, check_finite=True)
    R = dfac.rank
    rows = shard.shape.dims[mode]
    prow = comm.padded(rows) if owner_rows else rows
    out = t.empty((prow, nat.padded_ld(R)), dtype=t.float64, device=nat.device())
    L = nat.layout_struct(shard.layout)
    bounds = lo = None
    nseg = acc = priv = 0
    if kernel == "segment" and shard.nnz > 0:
        plan = segment_plan(shard, mode, R)
        d = plan["segments"]._dev
        bounds, lo, nseg, acc = nat.ptr(d["bounds"]), nat.ptr(d["lo"]), plan["L"], plan["acc_rows"]
        priv = int(plan["smem_bytes"] <= _smem_limit())
    elif kernel not in ("segment", "atomic"):
        raise ValueError(f"kernel must be 'segment' or 'atomic', not {kernel!r}")
    nat.call("alto_mttkrp_sharded", ctypes.byref(L), nat.ptr(shard._keys), nat.ptr(shard._vals), shard.nnz,
             ctypes.byref(dfac.struct), mode, nat.ptr(out), out.stride(0), rows, bounds, lo, nseg, acc, priv,
             int(owner_rows), comm.comm, nat.stream_ptr())
    return out


def _smem_limit() -> int:
    from .kernels import _smem_optin

    return _smem_optin()
