"""MTTKRP over the device-resident ALTO tensor, with the reference's strategy
API and a GPU-side adaptive kernel choice.

Public surface and decision rules restate pkg/src/alto/kernels.py:
``Strategy``/``StrategyChoice`` (:46-74), ``select_strategy`` (:77-119),
``resolve_strategy`` (:306-346), the three strategy entry points
(:160-252), ``mttkrp_with_choice``/``mttkrp`` (:255-303) and
``flops_per_nonzero`` (:349-351).

Two execution modes, both on the GPU (there is no CPU path):

* exact (``exact=True`` or ``ALTO_B200_EXACT=1``): each strategy runs the
  reference's own accumulation order -- sequential and recursive through
  per-segment private buffers + ascending pull reduction, output-oriented
  through register row runs + ascending boundary merge -- with no FMA
  contraction, so results are bit-identical to the reference for the same
  number of segments.
* fast (default): the GPU picks its kernel per mode (``select_gpu_kernel``):
  the output-oriented register-run kernel over a cached mode-ordered copy of
  the stream, or direct fp64 reductions over the ALTO stream itself.
  Results agree with the reference to ~1e-15 relative.
"""

from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .partition import (
    ModeOrderedView,
    SegmentSet,
    balanced_bounds,
    device_dview,
    device_fused_stream,
    device_mode_view,
    make_mode_ordered_view,
    make_segments,
)
from .tensor import AltoTensor, TensorStats, compute_stats
from .validation import check_factors, check_finite_device, check_mode

DEFAULT_TEMP_BUDGET_BYTES = 1 << 30

REUSE_THRESHOLD = 4.0

GPU_KERNELS = ("dview", "oriented", "atomic", "segment", "segment-atomic")


class Strategy(enum.Enum):
    SEQUENTIAL = "sequential"
    RECURSIVE = "recursive"
    OUTPUT_ORIENTED = "output"


@dataclass(frozen=True)
class StrategyChoice:
    strategy: Strategy
    mode: int
    workers: int
    fiber_reuse: float
    buffer_bytes: int | None
    temp_budget_bytes: int
    reason: str
    kernel: str = ""
    kernel_reason: str = ""

    def to_json_dict(self) -> dict:
        # identical record to the reference (workers deliberately omitted)
        return {
            "strategy": self.strategy.value,
            "mode": self.mode,
            "fiber_reuse": self.fiber_reuse,
            "buffer_bytes": self.buffer_bytes,
            "temp_budget_bytes": self.temp_budget_bytes,
            "reason": self.reason,
        }

    def gpu_json_dict(self) -> dict:
        return {"mode": self.mode, "kernel": self.kernel, "reason": self.kernel_reason}


def select_strategy(stats: TensorStats, mode: int, workers: int, buffer_bytes: int | None = None,
                    temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES) -> StrategyChoice:
    """Reference rule: one worker -> sequential; reuse <= 4 -> output
    oriented; buffers over budget -> output oriented; else recursive."""
    check_mode(mode, stats.shape.ndim)
    reuse = stats.fiber_reuse[mode]

    def choice(strategy, reason):
        return StrategyChoice(strategy, mode, workers, reuse, buffer_bytes, temp_budget_bytes, reason)

    if workers <= 1:
        return choice(Strategy.SEQUENTIAL, "single worker")
    if reuse <= REUSE_THRESHOLD:
        return choice(Strategy.OUTPUT_ORIENTED, f"fiber reuse {reuse:.3g} <= {REUSE_THRESHOLD:g}")
    if buffer_bytes is not None and buffer_bytes > temp_budget_bytes:
        return choice(Strategy.OUTPUT_ORIENTED,
                      f"segment buffers need {buffer_bytes} bytes > budget {temp_budget_bytes}")
    return choice(Strategy.RECURSIVE, f"fiber reuse {reuse:.3g} > {REUSE_THRESHOLD:g}")


def resolve_strategy(alto: AltoTensor, mode: int, workers: int, rank: int, num_segments: int,
                     strategy="auto", temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES,
                     ) -> StrategyChoice:
    key = ("choice", mode, workers, rank, num_segments, str(strategy), temp_budget_bytes,
           os.environ.get("ALTO_B200_KERNEL", ""))
    hit = alto._cache.get(key)
    if hit is not None:
        return hit
    alto._cache[key] = choice = _resolve_strategy(alto, mode, workers, rank, num_segments, strategy,
                                                  temp_budget_bytes)
    return choice


def _resolve_strategy(alto: AltoTensor, mode: int, workers: int, rank: int, num_segments: int,
                      strategy, temp_budget_bytes: int) -> StrategyChoice:
    if isinstance(strategy, Strategy):
        strategy = strategy.value
    if strategy == "seq":
        strategy = "sequential"
    stats = compute_stats(alto)
    if strategy == "auto":
        reuse = stats.fiber_reuse[mode]
        buffer_bytes = None
        if workers > 1 and reuse > REUSE_THRESHOLD:
            buffer_bytes = make_segments(alto, num_segments).buffer_bytes(mode, rank)
        base = select_strategy(stats, mode, workers, buffer_bytes=buffer_bytes,
                               temp_budget_bytes=temp_budget_bytes)
    else:
        try:
            explicit = Strategy(strategy)
        except ValueError:
            raise ValueError(
                f"strategy must be 'auto' or one of {[s.value for s in Strategy]}, got {strategy!r}"
            ) from None
        base = StrategyChoice(explicit, mode, workers, stats.fiber_reuse[mode], None,
                              temp_budget_bytes, "explicit request")
    kernel, why = select_gpu_kernel(alto, mode, rank, base.strategy)
    return StrategyChoice(base.strategy, base.mode, base.workers, base.fiber_reuse, base.buffer_bytes,
                          base.temp_budget_bytes, base.reason, kernel, why)


def select_gpu_kernel(alto: AltoTensor, mode: int, rank: int, strategy: Strategy):
    """GPU analogue of the paper's adaptive conflict resolution (per mode;
    the reference's rule is pkg/src/alto/kernels.py:77-119 and stays recorded
    unchanged in ``StrategyChoice``). Candidates, in the order the measured
    B200 numbers rank them (profiles/r02_segment_ab.md):

    1. ``dview`` -- privatise every output row in registers over a decoded,
       mode-ordered copy of the stream (20 B/nnz for 3 modes; row runs
       average ``fiber_reuse`` = nnz / I_n nonzeros and are written once).
       Wins every BASELINE mode it can run on: c2 1.18 ms vs 8.3 (segment
       kernel without privatisation) and 7.0 (atomics); c3 mode 3 5.9 ms vs
       12.6 (segment kernel, interval in shared memory). On a 3-mode tensor
       of rank <= 32 the copy is the interleaved (row, next-mode) fiber
       stream and the kernel the fused fiber-factored one
       (csrc/memo_sums.cu: the next mode's row once per fiber; c2 0.90 ms).
    2. ``segment`` -- the paper's kernel: one CTA per ALTO line segment, the
       segment's output interval privatised in shared memory, no copy of the
       stream. Needs the widest interval x R x 8 B to fit (fiber reuse high
       enough that a short mode's rows fit on chip: c3 mode 3, 168 rows;
       c5 mode 4, 1000 rows). Chosen when the decoded copy does not fit in
       device memory: c5 mode 4 99 ms vs 1356 ms with atomics.
    3. ``atomic`` -- fp64 reductions straight from the ALTO stream (always
       possible; L2-atomic bound).

    ``ALTO_B200_KERNEL`` forces a kernel (benchmarks, tests)."""
    forced = os.environ.get("ALTO_B200_KERNEL", "").strip().lower()
    if forced in GPU_KERNELS:
        return forced, "forced by ALTO_B200_KERNEL"
    reuse = alto.nnz / alto.shape.dims[mode]
    # decoded views need coordinates < 2^32 and 2..5 modes; a 2-mode tensor
    # takes the key view (same register row runs, keys decoded in registers)
    dview_ok = 2 <= alto.ndim <= 5 and max(alto.shape.dims) < 2**32
    kind = "dview" if dview_ok else "oriented"
    why = ("register row runs over a decoded mode-ordered copy" if dview_ok
           else "register row runs over a mode-ordered key copy")
    if dview_ok and _use_fused(alto, rank):
        why = (f"register row runs over the interleaved (row, mode {_fused_fiber_mode(alto, mode)}) fiber stream, "
               "that mode's row once per fiber (fused fiber kernel)")
    if ("dview" if dview_ok else "view", mode) in alto._cache or any(
            isinstance(k, tuple) and k[:2] == ("fstream", mode) for k in alto._cache):
        return kind, f"fiber reuse {reuse:.3g}: mode-ordered copy cached; {why}"
    key_bytes = 8 if alto.layout.word_bits == 64 else 16
    need = alto.nnz * (key_bytes + 16) * 2  # the copy + sort scratch while it is built
    try:
        free = nat.torch().cuda.mem_get_info()[0]
    except Exception:
        free = need
    if need <= 0.8 * free:
        return kind, f"fiber reuse {reuse:.3g}: mode-ordered copy ({need / 2e9:.2f} GB) fits; {why}"
    # no room for a copy: privatise the ALTO segments' intervals on chip when
    # they fit (a short mode: high fiber reuse), else reduce directly
    if 3 <= alto.ndim <= 5 and max(alto.shape.dims) < 2**32:
        plan = segment_plan(alto, mode, rank)
        if plan["smem_bytes"] <= _smem_optin():
            return "segment", (f"fiber reuse {reuse:.3g}, widest segment interval {plan['acc_rows']} rows "
                               f"({plan['smem_bytes'] / 1024:.0f} KB) fits in shared memory; mode-ordered copy "
                               f"({need / 2e9:.2f} GB) does not fit: ALTO line segments, privatised")
        return "atomic", (f"fiber reuse {reuse:.3g}: neither a mode-ordered copy ({need / 2e9:.2f} GB) nor the "
                          f"segment intervals ({plan['acc_rows']} rows) fit: direct fp64 reductions")
    return "atomic", f"mode-ordered copy ({need / 2e9:.2f} GB) exceeds free memory: direct fp64 reductions"


def _smem_optin() -> int:
    try:
        return int(nat.torch().cuda.get_device_properties(nat.device()).shared_memory_per_block_optin)
    except Exception:
        return 227 * 1024


def resolve_exact(exact) -> bool:
    if exact is None:
        return nat.env_flag("ALTO_B200_EXACT", False)
    return bool(exact)


# ---------------------------------------------------------------------------
# device launch helpers shared with cpd.apr


class DeviceFactors:
    """Factor matrices staged on the device with 32-byte aligned rows.

    ``check_finite``: scan the uploaded factors for non-finite entries on the
    device (``alto_factors_nonfinite``) -- the finiteness part of
    check_factors (pkg/src/alto/validation.py:30-57). With ``defer`` the
    flags stay on the device and ``verify`` (or ``_finish``, which reads them
    back with the result) raises later, so the upload, the scan and the
    kernel that consumes the factors are queued without a host round trip;
    a non-finite input still raises before any result is returned."""

    def __init__(self, factors, rank: int | None = None, *, check_finite: bool = False, skip: int = -1,
                 defer: bool = False, staging: dict | None = None):
        """``skip``: a mode whose factor the launch does not read (the MTTKRP
        target): it is validated on the host and not uploaded. ``staging``:
        a dict (the tensor's cache) whose device buffers, flag buffer and
        factor struct are reused across calls -- only for host inputs of
        calls that synchronise before returning (the public numpy path), so
        a buffer is never refilled while a kernel still reads it."""
        t = nat.torch()
        self.rank = int(rank if rank is not None else factors[0].shape[1])
        self.flags = None
        self._skip_bad = False
        self._skip_src = None  # target factor awaiting its host scan (deferred)
        ld = nat.padded_ld(self.rank)
        N = len(factors)
        if staging is not None and 8 * ld * sum(int(f.shape[0]) for f in factors) > (256 << 20):
            staging = None  # large factors: no persistent copies
        shape_key = ("stage", self.rank, skip, tuple(int(f.shape[0]) for f in factors))
        hit = staging.get(shape_key) if staging is not None else None
        uploaded = False
        if hit is not None:
            mats, struct, flags, rows = hit
            if not any(isinstance(f, t.Tensor) for f in factors):
                # contiguous (rows, rank) numpy factors: copies + finiteness
                # scan in one C call (alto_upload_factors)
                hp = (ctypes.c_void_p * N)(*[None if n == skip else f.ctypes.data for n, f in enumerate(factors)])
                nat.call("alto_upload_factors", ctypes.byref(struct), hp, rows, self.rank, int(skip),
                         ctypes.c_void_p(flags.data_ptr()) if check_finite else None, nat.stream_ptr())
                uploaded = True
            else:
                for n, f in enumerate(factors):
                    if n != skip:
                        src = f if isinstance(f, t.Tensor) else t.from_numpy(f)
                        mats[n][:, : self.rank].copy_(src, non_blocking=True)
        else:
            mats = []
            for n, f in enumerate(factors):
                if n == skip:
                    mats.append(t.zeros((1, ld), dtype=t.float64, device=nat.device()))
                else:
                    mats.append(nat.to_device_matrix(f, non_blocking=True))
            struct = nat.factors_struct(mats, self.rank)
            flags = t.empty(N, dtype=t.int32, device=nat.device())
            rows = (ctypes.c_int64 * N)(*[0 if n == skip else int(m.shape[0]) for n, m in enumerate(mats)])
            if staging is not None:
                staging[shape_key] = (mats, struct, flags, rows)
        if check_finite and skip >= 0:
            self._skip_src = factors[skip]
        self.mats = mats
        self.struct = struct
        if check_finite:
            self.flags = flags
            if not uploaded:
                nat.call("alto_factors_nonfinite", ctypes.byref(self.struct), rows, int(skip),
                         ctypes.c_void_p(self.flags.data_ptr()), nat.stream_ptr())
            self.skip = skip
            if not defer:
                self.verify()

    def host_checks(self) -> None:
        """Scan the (not uploaded) target factor on the host; with ``defer``
        the caller runs this while the device works."""
        if self._skip_src is not None:
            self._skip_bad = not _host_all_finite(self._skip_src)
            self._skip_src = None

    def verify(self, host_flags=None) -> None:
        """Raise the reference's error for the lowest non-finite mode."""
        if self.flags is None:
            return
        self.host_checks()
        flags = list(host_flags if host_flags is not None else self.flags.cpu().tolist())
        if self._skip_bad:
            flags[self.skip] = 1
        for n, bad in enumerate(flags):
            if bad:
                raise ValueError(f"factor {n} contains non-finite entries")


def _host_all_finite(a) -> bool:
    """All entries finite: one vectorised sum (non-finite iff some entry is,
    barring overflow), with the exact scan only when the sum is not finite."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.size == 0 or np.isfinite(np.add.reduce(arr, axis=None)):
        return True
    return bool(np.isfinite(arr).all())


def _zeros_out(rows: int, rank: int):
    t = nat.torch()
    return t.zeros((rows, nat.padded_ld(rank)), dtype=t.float64, device=nat.device())


def _exact_segments(alto: AltoTensor, L: int, mode: int, rank: int):
    """Segment tables + zeroed packed temps for the exact recursive kernels."""
    t = nat.torch()
    segs = make_segments(alto, L)
    lo, hi = segs._dev["lo"], segs._dev["hi"]
    widths = (hi[:, mode] - lo[:, mode] + 1) * rank
    offs = t.zeros_like(widths)
    if widths.numel() > 1:
        offs[1:] = t.cumsum(widths, 0)[:-1]
    total = int(widths.sum())
    temps = t.zeros(max(total, 1), dtype=t.float64, device=nat.device())
    return segs, offs.contiguous(), temps


def launch_mttkrp(alto: AltoTensor, dfac: DeviceFactors, mode: int, kernel: str, *,
                  num_segments: int = 1, out=None):
    """Run one MTTKRP on the device. kernel: 'exact-seq' | 'exact-rec' |
    'exact-output' | 'oriented' | 'atomic'. Returns the (I, ld) device output."""
    t = nat.torch()
    R = dfac.rank
    rows = alto.shape.dims[mode]
    st = nat.stream_ptr()
    if out is None:
        out = _zeros_out(rows, R)
    elif out.is_contiguous():
        nat.call("alto_memset_async", nat.ptr(out), out.numel() * out.element_size(), st)
    else:
        out.zero_()
    L = nat.layout_struct(alto.layout)
    M = alto.nnz
    if kernel in ("exact-seq", "exact-rec"):
        nseg = 1 if kernel == "exact-seq" else min(num_segments, M)
        segs, offs, temps = _exact_segments(alto, nseg, mode, R)
        d = segs._dev
        nat.call("alto_mttkrp_exact", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(out), out.stride(0), nat.ptr(d["bounds"]),
                 nat.ptr(d["lo"]), nat.ptr(d["hi"]), nat.ptr(offs), nseg, nat.ptr(temps), st)
    elif kernel in ("exact-output", "oriented"):
        _perm, vkeys, vvals = device_mode_view(alto, mode)
        exact = kernel == "exact-output"
        nseg = min(num_segments, M) if exact else nat.default_segments(M)
        scratch = _run_scratch(alto, nseg)
        nat.call("alto_mttkrp_oriented", ctypes.byref(L), nat.ptr(vkeys), nat.ptr(vvals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(out), out.stride(0), nseg, int(exact),
                 nat.ptr(scratch), scratch.numel(), st)
    elif kernel == "dview" and _use_fused(alto, R):
        # the fiber-factored branch-free kernel over the interleaved (row,
        # fiber) stream: the fiber mode's row once per fiber, the other N - 2
        # per nonzero (csrc/memo_sums.cu); with 3 modes the memoised sweep's
        # producer stream without the piece sums (same fiber mode, shared)
        fm = _fused_fiber_mode(alto, mode)
        fr, fj, fk, fv = device_fused_stream(alto, mode, fm, R)
        aj = dfac.mats[fm]
        others = [m for m in range(alto.ndim) if m not in (mode, fm)]
        aks = (ctypes.c_void_p * 3)(*[dfac.mats[m].data_ptr() for m in others])
        lds = (ctypes.c_int64 * 3)(*[dfac.mats[m].stride(0) for m in others])
        nat.call("alto_mttkrp_fused", nat.ptr(fr), nat.ptr(fj), nat.ptr(fk), nat.ptr(fv), M, len(others),
                 nat.ptr(aj), aj.stride(0), ctypes.cast(aks, ctypes.c_void_p), ctypes.cast(lds, ctypes.c_void_p), R,
                 nat.ptr(out), out.stride(0), st)
    elif kernel == "dview":
        fm, rows, crd, vvals, recur = device_dview(alto, mode, R)
        nat.call("alto_mttkrp_dview", ctypes.byref(L), nat.ptr(rows), nat.ptr(crd), nat.ptr(vvals), M,
                 ctypes.byref(dfac.struct), mode, int(recur), -1,
                 nat.ptr(out), out.stride(0), st)
    elif kernel in ("segment", "segment-atomic"):
        plan = segment_plan(alto, mode, R)
        d = plan["segments"]._dev
        nat.call("alto_mttkrp_segment", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(out), out.stride(0), nat.ptr(d["bounds"]),
                 nat.ptr(d["lo"]), plan["L"], plan["acc_rows"], int(kernel == "segment"), st)
    elif kernel == "atomic":
        nat.call("alto_mttkrp_stream", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(out), out.stride(0), nat.ALGO_ATOMIC,
                 None, None, 0, st)
    else:
        raise ValueError(f"unknown GPU kernel {kernel!r}")
    return out




def _use_fused(alto: AltoTensor, rank: int) -> bool:
    """MTTKRP of rank <= 32 through the fused fiber kernel for 3 and 4 modes
    (c2 0.90 vs 1.17 ms per mode for dview3, c3 22.2 vs 23.5 ms per sweep);
    5 modes stay on dview3 (c5 201 vs 146 ms per sweep, profiles/
    r02_fused_nmode_ab.txt) unless ALTO_B200_FUSED_MODES=5.
    ALTO_B200_FUSED=0 keeps dview3 everywhere; deterministic mode keeps
    dview3's ordered edge merge."""
    top = int(nat.env_str("ALTO_B200_FUSED_MODES", "4") or 4)
    return (3 <= alto.ndim <= min(top, 5) and rank <= 32 and max(alto.shape.dims) < 2**30
            and not nat.deterministic() and nat.env_flag("ALTO_B200_FUSED", True))


def _fused_fiber_mode(alto: AltoTensor, mode: int) -> int:
    """The fused kernel's fiber mode: with 3 modes the next mode (the
    memoised sweep's producer stream, shared), else the longest other mode
    (its rows are the ones that miss L2; c3 modes 0-2: 5.39 vs 5.47 ms per
    mode with the shortest, `profiles/r02_fused_fiber_choice_ab.txt`,
    although the shortest gives longer fibers: 5.6 vs 2.7 nonzeros,
    `profiles/r02_fiber_stats.jsonl`). ALTO_B200_FUSED_FIBER=short|long|<mode>
    overrides."""
    if alto.ndim == 3:
        return (mode + 1) % 3
    dims = alto.shape.dims
    pick = nat.env_str("ALTO_B200_FUSED_FIBER", "long").lower()
    others = [m for m in range(alto.ndim) if m != mode]
    if pick.isdigit() and int(pick) in others:
        return int(pick)
    if pick == "short":
        return min(others, key=lambda m: (dims[m], m))
    return max(others, key=lambda m: (dims[m], -m))


def segment_count(alto: AltoTensor) -> int:
    """Line segments (one CTA each, one resident CTA per SM) of the ALTO
    segment kernel: ``ALTO_B200_SEG_WAVES`` waves of the SM count."""
    waves = max(int(os.environ.get("ALTO_B200_SEG_WAVES", "2")), 1)
    return max(1, min(alto.nnz, nat.sm_count() * waves))


def segment_plan(alto: AltoTensor, mode: int, rank: int) -> dict:
    """Segments and accumulator size of the ALTO line-segment kernel for one
    mode: L balanced segments (``make_segments``, the reference's
    partition.py:78-123), the widest interval of the mode (rows of the
    shared-memory accumulator) and the shared memory that needs."""
    L = segment_count(alto)
    key = ("segplan", mode, rank, L)
    plan = alto._cache.get(key)
    if plan is None:
        segs = make_segments(alto, L)
        widths = [s.interval_width(mode) for s in segs.segments]
        acc_rows = max(widths)
        nb = ctypes.c_size_t(0)
        nat.call("alto_segment_smem_bytes", alto.layout.word_bits, alto.ndim, rank, acc_rows, ctypes.byref(nb))
        plan = {"L": len(segs.segments), "segments": segs, "acc_rows": acc_rows, "smem_bytes": nb.value,
                "mean_width": sum(widths) / len(widths)}
        alto._cache[key] = plan
    return plan


def _run_scratch(alto: AltoTensor, nseg: int):
    key = ("run_scratch", nseg)
    s = alto._cache.get(key)
    if s is None:
        s = nat.run_scratch(nseg)
        alto._cache[key] = s
    return s


def kernel_for(choice: StrategyChoice, exact: bool) -> str:
    if exact:
        return {
            Strategy.SEQUENTIAL: "exact-seq",
            Strategy.RECURSIVE: "exact-rec",
            Strategy.OUTPUT_ORIENTED: "exact-output",
        }[choice.strategy]
    return choice.kernel or "oriented"


def _returns_torch(factors) -> bool:
    return any(type(f).__module__.startswith("torch") for f in factors)


def _finish(out, rank: int, as_torch: bool, dfac: "DeviceFactors | None" = None, extra=None, on_sync=None):
    """``extra``: a small device int32 tensor read back with the result
    (host numpy path), handed to ``on_sync`` after the stream sync."""
    res = out[:, :rank]
    if as_torch:
        if dfac is not None:
            dfac.verify()
        return res
    # D2H of the result (and of deferred finiteness flags) into pinned memory,
    # one stream sync; the numpy array keeps the buffer alive
    t = nat.torch()
    host = t.empty(tuple(res.shape), dtype=res.dtype, pin_memory=True)
    host.copy_(res, non_blocking=True)
    hflags = None
    if dfac is not None and dfac.flags is not None:
        hflags = t.empty(dfac.flags.shape, dtype=t.int32, pin_memory=True)
        hflags.copy_(dfac.flags, non_blocking=True)
    hextra = None
    if extra is not None:
        hextra = t.empty(extra.shape, dtype=extra.dtype, pin_memory=True)
        hextra.copy_(extra, non_blocking=True)
    if dfac is not None:
        dfac.host_checks()  # overlaps the queued device work
    t.cuda.current_stream().synchronize()
    if on_sync is not None:
        on_sync(hextra.tolist() if hextra is not None else None)
    if dfac is not None:
        dfac.verify(None if hflags is None else hflags.tolist())
    return host.numpy()


def _prepare(alto: AltoTensor, factors, mode: int):
    """Shape checks on the host; numpy factors are checked for finiteness
    on the device after their upload (DeviceFactors(check_finite=True))."""
    host = not _returns_torch(factors)
    factors = check_factors(factors, alto.shape, finite=not host)
    check_mode(mode, alto.ndim)
    return factors, factors[0].shape[1]


def _explicit(alto, factors, mode, strategy: Strategy, num_segments: int, exact):
    factors, rank = _prepare(alto, factors, mode)
    exact = resolve_exact(exact)
    kernel = kernel_for(StrategyChoice(strategy, mode, 1, 0.0, None, 0, "",
                                       *select_gpu_kernel(alto, mode, rank, strategy)), exact)
    host_in = not _returns_torch(factors)
    dfac = DeviceFactors(factors, rank, check_finite=host_in, defer=host_in)
    out = launch_mttkrp(alto, dfac, mode, kernel, num_segments=num_segments)
    return _finish(out, rank, not host_in, dfac if host_in else None)


def mttkrp_sequential(alto: AltoTensor, factors, mode: int, *, exact=None):
    """Sequential strategy (pkg/src/alto/kernels.py:160-166)."""
    return _explicit(alto, factors, mode, Strategy.SEQUENTIAL, 1, exact)


def mttkrp_recursive(alto: AltoTensor, segments: SegmentSet, factors, mode: int, workers: int = 1,
                     *, exact=None):
    """Recursive (buffered) strategy with the given segments
    (pkg/src/alto/kernels.py:169-184)."""
    return _explicit(alto, factors, mode, Strategy.RECURSIVE, segments.num_segments, exact)


def mttkrp_output_oriented(alto: AltoTensor, view: ModeOrderedView, factors, mode: int,
                           workers: int = 1, *, exact=None):
    """Output-oriented strategy over a mode-ordered view
    (pkg/src/alto/kernels.py:213-229)."""
    if view.mode != mode:
        raise ValueError(f"view is ordered by mode {view.mode}, not {mode}")
    return _explicit(alto, factors, mode, Strategy.OUTPUT_ORIENTED, view.num_segments, exact)


def mttkrp_with_choice(alto: AltoTensor, factors, mode: int, *, workers: int = 1,
                       num_segments: int | None = None, strategy="auto",
                       temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES, exact=None,
                       device_factors: DeviceFactors | None = None, out=None):
    factors, rank = _prepare(alto, factors, mode)
    num_segments = num_segments if num_segments is not None else max(workers, 1)
    choice = resolve_strategy(alto, mode, workers, rank, num_segments, strategy, temp_budget_bytes)
    kernel = kernel_for(choice, resolve_exact(exact))
    # the target mode's factor is not read by any MTTKRP kernel: numpy inputs
    # validate it on the host and skip its upload
    host_in = not _returns_torch(factors)
    dfac = device_factors if device_factors is not None else DeviceFactors(
        factors, rank, check_finite=host_in, skip=mode if host_in else -1, defer=host_in,
        staging=alto._cache if host_in else None)
    if out is None and host_in:
        # the device output is only read back (synchronised) before the call
        # returns: one buffer per (mode, rank) is reused across calls
        okey = ("out", mode, rank)
        out = alto._cache.get(okey)
        if out is None:
            out = alto._cache[okey] = _zeros_out(alto.shape.dims[mode], rank)
    if host_in and device_factors is None and alto.ndim == 3:
        # a user's CP-ALS loop through this call: the memoised dimension-tree
        # reuse across calls (memo.CallMemo), decided on the device
        from .memo import call_memo

        cm = call_memo(alto, rank)
        if cm is not None and cm.observe(mode) and kernel == "dview" and _use_fused(alto, rank):
            cm.launch(dfac, mode, out)
            res = _finish(out, rank, False, dfac, extra=cm.flag, on_sync=lambda f: cm.settle(bool(f[0])))
            return res, choice
    dout = launch_mttkrp(alto, dfac, mode, kernel, num_segments=num_segments, out=out)
    return _finish(dout, rank, not host_in, dfac if device_factors is None and host_in else None), choice


def mttkrp(alto: AltoTensor, factors, mode: int, *, workers: int = 1, num_segments: int | None = None,
           strategy="auto", temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES, exact=None):
    out, _ = mttkrp_with_choice(alto, factors, mode, workers=workers, num_segments=num_segments,
                                strategy=strategy, temp_budget_bytes=temp_budget_bytes, exact=exact)
    return out


def flops_per_nonzero(ndim: int, rank: int) -> int:
    return 2 * rank * (ndim - 1) + rank
