"""Balanced line segments and mode-ordered views, computed on the GPU.

Restates pkg/src/alto/partition.py: ``balanced_bounds`` (:69-75) is host
arithmetic; the per-segment interval reduction (:91-95), boundary-row flags
(:117-120, :126-134) and the stable per-mode sort of the view (:185-199) run
as device kernels. Results are cached on the tensor exactly like the
reference (``_segments`` per L, ``_views`` per (mode, L)); the device copies
used by the kernels ride along.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .encoding import position_to_int
from .tensor import AltoTensor, device_decode


@dataclass(frozen=True)
class Segment:
    start: int
    stop: int
    pos_first: int
    pos_last: int
    intervals: tuple[tuple[int, int], ...]

    @property
    def size(self) -> int:
        return self.stop - self.start

    def interval_width(self, mode: int) -> int:
        lo, hi = self.intervals[mode]
        return hi - lo + 1


class SegmentSet:
    """All segments plus per-mode boundary rows (rows in >= 2 segments).

    Boundary rows are computed lazily per mode on first access (one device
    pass per mode), since the kernels only need the intervals."""

    def __init__(self, segments, alto: AltoTensor, dev: dict):
        self.segments = tuple(segments)
        self._alto = alto
        self._dev = dev  # device bounds/lo/hi tensors
        self._boundary = [None] * alto.ndim

    @property
    def num_segments(self) -> int:
        return len(self.segments)

    @property
    def boundary_rows(self) -> tuple[np.ndarray, ...]:
        return tuple(self.boundary_rows_of(n) for n in range(self._alto.ndim))

    def boundary_rows_of(self, mode: int) -> np.ndarray:
        if self._boundary[mode] is None:
            self._boundary[mode] = _rows_spanning_segments(self._alto, mode, self.num_segments,
                                                           self._dev["bounds"])
        return self._boundary[mode]

    def bounds(self) -> np.ndarray:
        edges = [s.start for s in self.segments]
        edges.append(self.segments[-1].stop)
        return np.asarray(edges, dtype=np.int64)

    def interval_arrays(self, mode: int) -> tuple[np.ndarray, np.ndarray]:
        lo = np.asarray([s.intervals[mode][0] for s in self.segments], dtype=np.int64)
        hi = np.asarray([s.intervals[mode][1] for s in self.segments], dtype=np.int64)
        return lo, hi

    def buffer_rows(self, mode: int) -> int:
        return sum(s.interval_width(mode) for s in self.segments)

    def buffer_bytes(self, mode: int, rank: int) -> int:
        return self.buffer_rows(mode) * rank * 8


def balanced_bounds(count: int, parts: int) -> np.ndarray:
    """``parts`` contiguous chunks whose sizes differ by at most one, the
    first ``count % parts`` getting the extra item."""
    base, extra = divmod(count, parts)
    idx = np.arange(parts + 1, dtype=np.int64)
    return idx * base + np.minimum(idx, extra)


def make_segments(alto: AltoTensor, num_segments: int) -> SegmentSet:
    if num_segments < 1:
        raise ValueError("need at least one segment")
    L = min(num_segments, alto.nnz)
    cached = alto._segments.get(L)
    if cached is not None:
        return cached
    t = nat.torch()
    dev = nat.device()
    N = alto.ndim
    bounds = t.empty(L + 1, dtype=t.int64, device=dev)
    lo = t.empty((L, N), dtype=t.int64, device=dev)
    hi = t.empty((L, N), dtype=t.int64, device=dev)
    nat.call("alto_partition", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             alto.nnz, L, nat.ptr(bounds), nat.ptr(lo), nat.ptr(hi), nat.stream_ptr())
    hb = bounds.cpu().numpy()
    hlo = lo.cpu().numpy()
    hhi = hi.cpu().numpy()
    # first/last positions of every segment (2L keys)
    idx = t.from_numpy(np.stack([hb[:-1], hb[1:] - 1], axis=1).reshape(-1)).to(dev)
    ends = alto._keys.index_select(0, idx).cpu().numpy().view(np.uint64)
    segments = []
    for l in range(L):
        if ends.ndim == 1:
            first, last = int(ends[2 * l]), int(ends[2 * l + 1])
        else:
            first, last = position_to_int(ends[2 * l]), position_to_int(ends[2 * l + 1])
        segments.append(Segment(
            start=int(hb[l]), stop=int(hb[l + 1]), pos_first=first, pos_last=last,
            intervals=tuple((int(a), int(b)) for a, b in zip(hlo[l], hhi[l])),
        ))
    # per-segment offsets into a packed temps buffer, per mode
    result = SegmentSet(segments, alto, {"bounds": bounds, "lo": lo, "hi": hi})
    alto._segments[L] = result
    return result


def _rows_spanning_segments(alto: AltoTensor, mode: int, L: int, dbounds) -> np.ndarray:
    t = nat.torch()
    dev = nat.device()
    I = alto.shape.dims[mode]
    rmin = t.empty(I, dtype=t.int32, device=dev)
    rmax = t.empty(I, dtype=t.int32, device=dev)
    nat.call("alto_row_segment_span", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             alto.nnz, mode, nat.ptr(dbounds), L, nat.ptr(rmin), nat.ptr(rmax), nat.stream_ptr())
    rows = t.nonzero((rmax >= 0) & (rmin != rmax)).reshape(-1)
    return rows.cpu().numpy().astype(np.int64)


def overlap(a: Segment, b: Segment, mode: int):
    lo = max(a.intervals[mode][0], b.intervals[mode][0])
    hi = min(a.intervals[mode][1], b.intervals[mode][1])
    return (lo, hi) if lo <= hi else None


class ModeOrderedView:
    """Nonzeros stably re-sorted by one mode (device resident).

    ``perm``/``coords``/``values`` are numpy views made on first access; the
    kernels read ``_keys``/``_vals`` (view order)."""

    def __init__(self, alto, mode, dperm, dkeys, dvals, bounds, boundary_rows):
        self.mode = mode
        self._alto = alto
        self._perm = dperm
        self._keys = dkeys
        self._vals = dvals
        self.bounds = bounds
        self.boundary_rows = boundary_rows
        self._np = {}

    @property
    def num_segments(self) -> int:
        return self.bounds.size - 1

    @property
    def perm(self) -> np.ndarray:
        if "perm" not in self._np:
            self._np["perm"] = self._perm.cpu().numpy()
        return self._np["perm"]

    @property
    def coords(self) -> np.ndarray:
        if "coords" not in self._np:
            self._np["coords"] = device_decode(self._alto.layout, self._keys).cpu().numpy()
        return self._np["coords"]

    @property
    def values(self) -> np.ndarray:
        if "values" not in self._np:
            self._np["values"] = self._vals.cpu().numpy()
        return self._np["values"]

    def boundary_slots(self, num_rows: int) -> np.ndarray:
        slots = np.full(num_rows, -1, dtype=np.int64)
        slots[self.boundary_rows] = np.arange(self.boundary_rows.size)
        return slots


def device_mode_view(alto: AltoTensor, mode: int):
    """Stable mode sort of the stream -> (perm, keys, vals) device tensors,
    cached per mode (independent of L)."""
    key = ("view", mode)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    dev = nat.device()
    M = alto.nnz
    perm = t.empty(M, dtype=t.int64, device=dev)
    vkeys = t.empty_like(alto._keys)
    vvals = t.empty_like(alto._vals)
    b = ctypes.c_size_t(0)
    nat.call("alto_mode_view_scratch_bytes", M, ctypes.byref(b))
    scratch = t.empty(b.value, dtype=t.uint8, device=dev)
    nat.call("alto_mode_view", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             nat.ptr(alto._vals), M, mode, nat.ptr(perm), nat.ptr(vkeys), nat.ptr(vvals),
             nat.ptr(scratch), b.value, nat.stream_ptr())
    del scratch
    alto._cache[key] = (perm, vkeys, vvals)
    return alto._cache[key]


# L1 budget for one factor's rows inside a block, and the shortest average
# (row, block) run for which blocking still pays (each run is flushed with an
# fp64 reduction instead of one plain store per row)
_BLOCK_L1_BYTES = 64 << 10
_BLOCK_MIN_RUN = 64.0


def view_plan(alto: AltoTensor, mode: int, rank: int = 16):
    """Order of the decoded view of ``mode`` -> (fiber_mode, block_mode,
    block_shift); -1 / 0 when unused.

    Rows are sub-sorted by the shortest other mode (fiber order: consecutive
    nonzeros share that factor row). When the largest remaining mode's factor
    exceeds the L1 budget and rows are long enough, the view is additionally
    cut into blocks of 2^shift of that mode's rows (outermost sort key), so
    the rows it gathers stay L1-resident while a block is walked; a row then
    recurs once per block. ``ALTO_B200_BLOCK=0`` disables blocking."""
    key = ("vplan", mode)
    if key in alto._cache:
        return alto._cache[key]
    dims = alto.shape.dims
    fm = fiber_mode_for(alto.shape, mode) if alto.ndim >= 3 else -1
    if os.environ.get("ALTO_B200_VIEW_ORDER", "").strip().lower() == "alto":
        # rows in ALTO order (stable sort by the row only): every gathered
        # mode keeps the linearisation's locality instead of one fiber mode
        alto._cache[("vplan", mode)] = (-1, -1, 0)
        return alto._cache[("vplan", mode)]
    others = [m for m in range(alto.ndim) if m not in (mode, fm)]
    bmode, shift = -1, 0
    if others and nat.env_flag("ALTO_B200_BLOCK", True):
        b = max(others, key=lambda m: (dims[m], -m))
        row_bytes = 8 * nat.padded_ld(rank)
        budget = int(os.environ.get("ALTO_B200_BLOCK_L1_BYTES", _BLOCK_L1_BYTES))
        shift = max((budget // row_bytes).bit_length() - 1, 0)
        nblocks = -(-dims[b] // (1 << shift))
        min_run = float(os.environ.get("ALTO_B200_BLOCK_MIN_RUN", _BLOCK_MIN_RUN))
        if nblocks > 1 and alto.nnz / (dims[mode] * nblocks) >= min_run:
            bmode = b
        else:
            shift = 0
    alto._cache[key] = (fm, bmode, shift)
    return alto._cache[key]


def prefer_unblocked(alto: AltoTensor, mode: int) -> None:
    """Fix the plan of a mode whose decoded view is not built yet to the
    unblocked fiber order. CP-APR does this: its Phi rereads one view many
    times (streamed-Pi iterations reduce every row run of a blocked view
    with atomics), and on c4 the gathering Phi is faster unblocked too
    (mode 2: 1.01 vs 1.15 ms; MTTKRP 0.85 vs 0.83 ms)."""
    if ("vplan", mode) in alto._cache or ("dview", mode) in alto._cache:
        return
    fm = fiber_mode_for(alto.shape, mode) if alto.ndim >= 3 else -1
    alto._cache[("vplan", mode)] = (fm, -1, 0)


def ensure_unblocked(alto: AltoTensor, mode: int) -> None:
    """Deterministic mode: a blocked view reduces every row run with fp64
    atomics, so drop a blocked plan (and its views) and fix the unblocked
    fiber order."""
    plan = alto._cache.get(("vplan", mode))
    if plan is not None and plan[1] >= 0:
        for key in (("dview", mode), ("bview", mode), ("vplan", mode)):
            alto._cache.pop(key, None)
    prefer_unblocked(alto, mode)


def device_blocked_view(alto: AltoTensor, mode: int, fm: int, bmode: int, shift: int):
    """Blocked fiber view -> (perm, keys, vals), cached."""
    key = ("bview", mode)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    dev = nat.device()
    M = alto.nnz
    perm = t.empty(M, dtype=t.int64, device=dev)
    vkeys = t.empty_like(alto._keys)
    vvals = t.empty_like(alto._vals)
    b = ctypes.c_size_t(0)
    nat.call("alto_mode_view_scratch_bytes", M, ctypes.byref(b))
    scratch = t.empty(b.value, dtype=t.uint8, device=dev)
    nat.call("alto_blocked_view", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             nat.ptr(alto._vals), M, mode, fm, bmode, shift, nat.ptr(perm), nat.ptr(vkeys), nat.ptr(vvals),
             nat.ptr(scratch), b.value, nat.stream_ptr())
    del scratch
    alto._cache[key] = (perm, vkeys, vvals)
    return alto._cache[key]


def _dview_source(alto: AltoTensor, mode: int, rank: int):
    """(cache key, perm, keys, vals, rows_recur) of the key view the decoded
    view is built from."""
    fm, bmode, shift = view_plan(alto, mode, rank)
    if bmode >= 0:
        perm, vkeys, vvals = device_blocked_view(alto, mode, fm, bmode, shift)
        return ("bview", mode), perm, vkeys, vvals, True
    if fm >= 0:
        _fm, perm, vkeys, vvals = device_fiber_view(alto, mode)
        return ("fview", mode), perm, vkeys, vvals, False
    perm, vkeys, vvals = device_mode_view(alto, mode)
    return ("view", mode), perm, vkeys, vvals, False


def device_dview(alto: AltoTensor, mode: int, rank: int = 16):
    """Decoded view for the fast output-oriented kernels -> (fiber_mode,
    rows, crd, vals, rows_recur), cached per mode.

    rows (u32) are the mode coordinates, crd (u32, SoA, row stride M rounded
    up to 8) the other modes' coordinates and vals the values, all in view
    order, planes in ascending mode order; the order is ``view_plan``'s
    (fiber sub-order, optionally blocked -- then ``rows_recur`` is True and
    the kernels reduce every row run). The key copy the view is decoded from
    is dropped again unless it was already cached."""
    if nat.deterministic():
        ensure_unblocked(alto, mode)
    key = ("dview", mode)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    M = alto.nnz
    skey = _dview_source_key(alto, mode, rank)
    had = skey in alto._cache
    _k, _perm, vkeys, vvals, recur = _dview_source(alto, mode, rank)
    rows = t.empty(M, dtype=t.int32, device=vkeys.device)
    # SoA block, row stride M rounded up to 8 (crd_stride in dview_kernels.cu)
    crd = t.empty((max(alto.ndim - 1, 1), (M + 7) & ~7), dtype=t.int32, device=vkeys.device)
    nat.call("alto_decode_view", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(vkeys), M, mode,
             nat.ptr(rows), nat.ptr(crd), nat.stream_ptr())
    fm = view_plan(alto, mode, rank)[0]
    alto._cache[key] = (fm, rows, crd, vvals, recur)
    if not had:
        del alto._cache[skey]
    return alto._cache[key]


def device_fused_stream(alto: AltoTensor, mode: int, fiber_mode: int, rank: int):
    """Interleaved fiber stream of ``mode`` sorted by (row, ``fiber_mode``
    coordinate), stable in ALTO order (csrc/memo_sums.cu layout: rows,
    j | piece start << 31 with j the fiber-mode coordinate, the N - 2 other
    modes' coordinates in ascending mode order as planes, values) -> (rows,
    jf, k planes, vals), cached per (mode, fiber mode, lanes per nonzero).
    3-5 modes, rank <= 32. The intermediate key copy and decoded view are
    freed."""
    N = alto.ndim
    if not 3 <= N <= 5 or fiber_mode == mode or not 0 <= fiber_mode < N:
        raise ValueError("fused streams need 3-5 modes and a fiber mode other than the row mode")
    g = 1
    while 4 * g < rank:
        g *= 2
    key = ("fstream", mode, fiber_mode, g)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    dev = nat.device()
    M = alto.nnz
    L = nat.layout_struct(alto.layout)
    perm = t.empty(M, dtype=t.int64, device=dev)
    b = ctypes.c_size_t(0)
    nat.call("alto_mode_view_scratch_bytes", M, ctypes.byref(b))
    scratch = t.empty(b.value, dtype=t.uint8, device=dev)
    st = nat.stream_ptr()
    if M > 0 and nat.env_str("ALTO_B200_STREAM_BUILD", "fused").lower() != "legacy":
        # sort + one pass (gather through the permutation, decode, interleave)
        n = ctypes.c_int64(0)
        nat.call("alto_il_length", M, rank, ctypes.byref(n))
        out = (t.empty(n.value, dtype=t.int32, device=dev), t.empty(n.value, dtype=t.int32, device=dev),
               t.empty((N - 2, n.value), dtype=t.int32, device=dev), t.empty(n.value, dtype=t.float64, device=dev))
        nat.call("alto_fused_stream_build", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M, mode,
                 fiber_mode, rank, nat.ptr(perm), nat.ptr(out[0]), nat.ptr(out[1]), nat.ptr(out[2]), nat.ptr(out[3]),
                 None, None, nat.ptr(scratch), b.value, st)
        alto._cache[key] = out
        return out
    # legacy three-pass build (permuted copy, decoded view, interleave)
    vkeys = t.empty_like(alto._keys)
    vvals = t.empty_like(alto._vals)
    nat.call("alto_fiber_view", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M, mode, fiber_mode,
             nat.ptr(perm), nat.ptr(vkeys), nat.ptr(vvals), nat.ptr(scratch), b.value, st)
    del scratch, perm
    rows = t.empty(M, dtype=t.int32, device=dev)
    crd = t.empty((N - 1, (M + 7) & ~7), dtype=t.int32, device=dev)
    nat.call("alto_decode_view", ctypes.byref(L), nat.ptr(vkeys), M, mode, nat.ptr(rows), nat.ptr(crd), st)
    del vkeys
    jplane = fiber_mode if fiber_mode < mode else fiber_mode - 1
    n = ctypes.c_int64(0)
    nat.call("alto_il_length", M, rank, ctypes.byref(n))
    out = (t.empty(n.value, dtype=t.int32, device=dev), t.empty(n.value, dtype=t.int32, device=dev),
           t.empty((N - 2, n.value), dtype=t.int32, device=dev), t.empty(n.value, dtype=t.float64, device=dev))
    nat.call("alto_fused_stream_n", nat.ptr(rows), nat.ptr(crd), crd.stride(0), N - 1, jplane, nat.ptr(vvals), M,
             rank, nat.ptr(out[0]), nat.ptr(out[1]), nat.ptr(out[2]), nat.ptr(out[3]), st)
    alto._cache[key] = out
    return out


def _dview_source_key(alto: AltoTensor, mode: int, rank: int):
    fm, bmode, _shift = view_plan(alto, mode, rank)
    return ("bview", mode) if bmode >= 0 else (("fview", mode) if fm >= 0 else ("view", mode))


def dview_order(alto: AltoTensor, mode: int, rank: int = 16):
    """(perm, keys) of the order device_dview's kernels walk (PRE rows)."""
    _k, perm, vkeys, _vals, _recur = _dview_source(alto, mode, rank)
    return perm, vkeys


def fiber_mode_for(shape, mode: int) -> int:
    """Second sort mode of a fiber view: the shortest other mode (most
    repeats per row; ties to the lower index). ``ALTO_B200_FIBER_ORDER=long``
    picks the longest instead (the shorter modes are then the ones gathered
    at random, a smaller working set)."""
    dims = shape.dims
    others = [m for m in range(len(dims)) if m != mode]
    if os.environ.get("ALTO_B200_FIBER_ORDER", "short").strip().lower() == "long":
        return max(others, key=lambda m: (dims[m], -m))
    return min(others, key=lambda m: (dims[m], m))


def device_fiber_view(alto: AltoTensor, mode: int):
    """Stream sorted by (mode coordinate, fiber-mode coordinate), stable in
    ALTO order inside a fiber -> (fiber_mode, perm, keys, vals), cached."""
    key = ("fview", mode)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    dev = nat.device()
    M = alto.nnz
    fm = fiber_mode_for(alto.shape, mode)
    perm = t.empty(M, dtype=t.int64, device=dev)
    vkeys = t.empty_like(alto._keys)
    vvals = t.empty_like(alto._vals)
    b = ctypes.c_size_t(0)
    nat.call("alto_mode_view_scratch_bytes", M, ctypes.byref(b))
    scratch = t.empty(b.value, dtype=t.uint8, device=dev)
    nat.call("alto_fiber_view", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             nat.ptr(alto._vals), M, mode, fm, nat.ptr(perm), nat.ptr(vkeys), nat.ptr(vvals),
             nat.ptr(scratch), b.value, nat.stream_ptr())
    del scratch
    alto._cache[key] = (fm, perm, vkeys, vvals)
    return alto._cache[key]


def make_mode_ordered_view(alto: AltoTensor, mode: int, num_segments: int) -> ModeOrderedView:
    if not 0 <= mode < alto.ndim:
        raise ValueError(f"mode {mode} out of range for {alto.ndim} modes")
    if num_segments < 1:
        raise ValueError("need at least one segment")
    L = min(num_segments, alto.nnz)
    key = (mode, L)
    cached = alto._views.get(key)
    if cached is not None:
        return cached
    t = nat.torch()
    perm, vkeys, vvals = device_mode_view(alto, mode)
    bounds = balanced_bounds(alto.nnz, L)
    cuts = bounds[1:-1]
    if cuts.size:
        idx = t.from_numpy(np.concatenate([cuts, cuts - 1])).to(vkeys.device)
        rows = device_decode(alto.layout, vkeys.index_select(0, idx))[:, mode].cpu().numpy()
        at, before = rows[: cuts.size], rows[cuts.size:]
        boundary = np.unique(at[at == before]).astype(np.int64)
    else:
        boundary = np.empty(0, dtype=np.int64)
    view = ModeOrderedView(alto, mode, perm, vkeys, vvals, bounds, boundary)
    alto._views[key] = view
    return view
