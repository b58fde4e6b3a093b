"""CP-APR multiplicative update with device-resident state.

Restates pkg/src/alto/cpd/apr.py: ``CpAprConfig``/``CpAprResult`` (:54-98),
``precompute_krp_rows`` (:101-111), ``phi_kernel`` (:114-180),
``kkt_violation`` (:183-185), ``select_krp_memory_mode`` (:188-197),
``poisson_loglik`` (:200-207) and ``cp_apr_mu`` (:210-346). The Phi kernel,
the Khatri-Rao rows, the fused KKT / ``b *= Phi`` epilogue and the
log-likelihood pass are sm_100a kernels; the per-mode bookkeeping (shift,
column sums, normalisation) is small I_n x R elementwise work on device.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from .. import _native as nat
from ..kernels import (
    DEFAULT_TEMP_BUDGET_BYTES,
    DeviceFactors,
    Strategy,
    StrategyChoice,
    _exact_segments,
    _returns_torch,
    _run_scratch,
    kernel_for,
    resolve_exact,
    resolve_strategy,
)
from ..partition import (device_dview, device_mode_view, dview_order,
                         prefer_unblocked)
from ..tensor import AltoTensor, TensorStats, compute_stats
from ..validation import (
    NumericalError,
    check_factors,
    check_mode,
    check_nonnegative_values,
    check_rank,
    check_workers,
)
from ..distributed import agree_kernels
from .model import KruskalModel, init_factors

DEFAULT_FAST_MEMORY_BYTES = 100 * (1 << 20)

_LOW_REUSE_BELOW = 5.0


@dataclass(frozen=True)
class CpAprConfig:
    rank: int = 16
    max_outer: int = 200
    max_inner: int = 10
    tau: float = 1e-4
    kappa: float = 1e-2
    kappa_tol: float = 1e-10
    eps: float = 1e-10
    memory_mode: str = "auto"
    fast_memory_bytes: int = DEFAULT_FAST_MEMORY_BYTES
    seed: int = 0
    workers: int = 1
    num_segments: int | None = None
    strategy: str = "auto"
    temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES
    track_inner_loglik: bool = False

    def __post_init__(self):
        check_rank(self.rank)
        check_workers(self.workers)
        if self.max_outer < 1 or self.max_inner < 1:
            raise ValueError("iteration caps must be >= 1")
        if min(self.tau, self.kappa, self.kappa_tol, self.eps) <= 0:
            raise ValueError("tau, kappa, kappa_tol, and eps must be positive")
        if self.memory_mode not in ("auto", "pre", "otf"):
            raise ValueError("memory_mode must be auto, pre, or otf")


@dataclass
class CpAprResult:
    model: KruskalModel
    kkt_trace: list
    inner_iters: list
    loglik_trace: list
    n_outer: int
    converged: bool
    memory_mode: str = "otf"
    strategies: list = field(default_factory=list)
    inner_loglik: list | None = None
    wall_time_s: float = 0.0

    @property
    def final_kkt(self) -> float:
        return max(self.kkt_trace[-1])


# ---------------------------------------------------------------------------
# device launches


def launch_pi(alto: AltoTensor, dfac: DeviceFactors, mode: int, keys=None):
    """Khatri-Rao rows for the given key stream (default: the ALTO order)."""
    t = nat.torch()
    keys = alto._keys if keys is None else keys
    ldp = nat.padded_ld(dfac.rank)
    pi = t.zeros((alto.nnz, ldp), dtype=t.float64, device=nat.device())
    nat.call("alto_pi", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(keys), alto.nnz,
             ctypes.byref(dfac.struct), mode, nat.ptr(pi), ldp, nat.stream_ptr())
    return pi


def launch_pi_dview(alto: AltoTensor, dfac: DeviceFactors, mode: int):
    """Khatri-Rao rows in the decoded view's order (PRE rows of the dview Phi)."""
    t = nat.torch()
    _fm, rows, crd, _vals, _recur = device_dview(alto, mode, dfac.rank)
    ldp = nat.padded_ld(dfac.rank)
    pi = t.zeros((alto.nnz, ldp), dtype=t.float64, device=nat.device())
    nat.call("alto_pi_dview", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(rows), nat.ptr(crd), alto.nnz,
             ctypes.byref(dfac.struct), mode, nat.ptr(pi), ldp, nat.stream_ptr())
    return pi


def launch_phi(alto: AltoTensor, dfac: DeviceFactors, mode: int, kernel: str, scaled, eps: float, *,
               pi=None, pi_view=None, num_segments: int = 1, out=None, skip=None, zero: bool = True,
               pi_il_out=None):
    """One Phi evaluation. ``scaled``: device (I, lds) matrix. ``pi``: Pi in
    ALTO order (exact-seq/exact-rec/atomic); ``pi_view``: Pi in view order
    (oriented kernels). ``skip``: device-driven inner-loop state (dview
    only): the zero-fill and the kernel are no-ops once that loop is done.
    ``pi_il_out`` (dview, on the fly): also store the Khatri-Rao rows in the
    streamed-Pi layout for ``launch_phi_pstream``."""
    t = nat.torch()
    R = dfac.rank
    rows = alto.shape.dims[mode]
    if skip is not None:
        if kernel != "dview" or out is None:
            raise ValueError("skip needs the dview kernel and an output buffer")
        if zero:
            nat.call("alto_zero_if", nat.ptr(out), out.stride(0), out.shape[0], nat.ptr(skip), nat.stream_ptr())
    elif out is None:
        out = t.zeros((rows, nat.padded_ld(R)), dtype=t.float64, device=nat.device())
    else:
        out.zero_()
    L = nat.layout_struct(alto.layout)
    st = nat.stream_ptr()
    M = alto.nnz
    lds = scaled.stride(0)
    if kernel in ("exact-seq", "exact-rec"):
        nseg = 1 if kernel == "exact-seq" else min(num_segments, M)
        segs, offs, temps = _exact_segments(alto, nseg, mode, R)
        d = segs._dev
        nat.call("alto_phi_exact", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(scaled), lds, nat.ptr(pi),
                 pi.stride(0) if pi is not None else 0, eps, nat.ptr(out), out.stride(0),
                 nat.ptr(d["bounds"]), nat.ptr(d["lo"]), nat.ptr(d["hi"]), nat.ptr(offs), nseg,
                 nat.ptr(temps), st)
    elif kernel in ("exact-output", "oriented"):
        _perm, vkeys, vvals = device_mode_view(alto, mode)
        exact = kernel == "exact-output"
        nseg = min(num_segments, M) if exact else nat.default_segments(M)
        scratch = _run_scratch(alto, nseg)
        nat.call("alto_phi_oriented", ctypes.byref(L), nat.ptr(vkeys), nat.ptr(vvals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(scaled), lds, nat.ptr(pi_view),
                 pi_view.stride(0) if pi_view is not None else 0, eps, nat.ptr(out), out.stride(0),
                 nseg, int(exact), nat.ptr(scratch), scratch.numel(), st)
    elif kernel == "dview":
        fm, rows_, crd, vvals, recur = device_dview(alto, mode, R)
        nat.call("alto_phi_dview", ctypes.byref(L), nat.ptr(rows_), nat.ptr(crd), nat.ptr(vvals), M,
                 ctypes.byref(dfac.struct), mode, int(recur), -1,
                 nat.ptr(scaled), lds, nat.ptr(pi_view),
                 pi_view.stride(0) if pi_view is not None else 0, eps, nat.ptr(out), out.stride(0),
                 nat.ptr(skip), nat.ptr(pi_il_out), st)
    elif pi_il_out is not None:
        raise ValueError("pi_il_out needs the dview kernel")
    elif kernel == "atomic":
        nat.call("alto_phi_stream", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M,
                 ctypes.byref(dfac.struct), mode, nat.ptr(scaled), lds, nat.ptr(pi),
                 pi.stride(0) if pi is not None else 0, eps, nat.ptr(out), out.stride(0),
                 nat.ALGO_ATOMIC, None, None, 0, st)
    else:
        raise ValueError(f"unknown GPU kernel {kernel!r}")
    return out


# ---------------------------------------------------------------------------
# streamed-Pi Phi (csrc/pstream.cu): inner iterations after the first of a
# mode stream the Khatri-Rao rows the first one stored instead of gathering


def pstream_sizes(alto: AltoTensor, rank: int):
    """(slots, Pi doubles) of the streamed-Pi layout."""
    slots, pid = ctypes.c_int64(0), ctypes.c_int64(0)
    nat.call("alto_pstream_sizes", alto.nnz, rank, ctypes.byref(slots), ctypes.byref(pid))
    return slots.value, pid.value


def _small_counts(alto: AltoTensor) -> bool:
    """Every value an integer in [0, 255] (count data): the streamed-Pi
    layout then stores u8 values (csrc/pstream.cu CMP), cached per tensor."""
    key = ("small_counts",)
    if key not in alto._cache:
        v = alto._vals
        alto._cache[key] = bool(((v >= 0) & (v <= 255) & (v == t_round(v))).all().item()) if v.numel() else False
    return alto._cache[key]


def t_round(v):
    return nat.torch().round(v)


def pstream_view(alto: AltoTensor, mode: int, rank: int):
    """The decoded view's rows/values in slot order, cached per mode ->
    (rows, values, compact): the compact layout (u16 rows, u8 values; 9
    fewer bytes per nonzero) when the mode has < 65536 rows and the values
    are small counts (ALTO_B200_PSTREAM_COMPACT=0 keeps u32 / f64)."""
    key = ("pstream", mode)
    if key in alto._cache:
        return alto._cache[key]
    t = nat.torch()
    _fm, rows, _crd, vvals, _recur = device_dview(alto, mode, rank)
    slots, _ = pstream_sizes(alto, rank)
    compact = (alto.shape.dims[mode] <= 65536 and _small_counts(alto)
               and nat.env_flag("ALTO_B200_PSTREAM_COMPACT", True))
    if compact:
        il_rows = t.empty(slots, dtype=t.int16, device=vvals.device)
        il_vals = t.empty(slots, dtype=t.uint8, device=vvals.device)
        nat.call("alto_pstream_build_compact", nat.ptr(rows), nat.ptr(vvals), alto.nnz, nat.ptr(il_rows),
                 nat.ptr(il_vals), nat.stream_ptr())
    else:
        il_rows = t.empty(slots, dtype=t.int32, device=vvals.device)
        il_vals = t.empty(slots, dtype=t.float64, device=vvals.device)
        nat.call("alto_pstream_build", nat.ptr(rows), nat.ptr(vvals), alto.nnz, nat.ptr(il_rows), nat.ptr(il_vals),
                 nat.stream_ptr())
    alto._cache[key] = (il_rows, il_vals, compact)
    return alto._cache[key]


def launch_phi_pstream(alto: AltoTensor, mode: int, rank: int, scaled, eps: float, pi_il, out, *, skip=None,
                       zero: bool = True):
    """Phi from streamed Khatri-Rao rows (``pi_il`` as stored by
    ``launch_phi(..., pi_il_out=...)`` with the same factors)."""
    if zero:
        if skip is not None:
            nat.call("alto_zero_if", nat.ptr(out), out.stride(0), out.shape[0], nat.ptr(skip), nat.stream_ptr())
        else:
            out.zero_()
    il_rows, il_vals, compact = pstream_view(alto, mode, rank)
    recur = device_dview(alto, mode, rank)[4]
    nat.call("alto_phi_pstream2", nat.ptr(il_rows), nat.ptr(il_vals), int(compact), nat.ptr(pi_il), alto.nnz, rank,
             int(recur),
             nat.ptr(scaled), scaled.stride(0), eps, nat.ptr(out), out.stride(0), nat.ptr(skip), nat.stream_ptr())
    return out


def apr_update(b, ratio, rank: int, tau: float, apply: int = -1):
    """Fused KKT + conditional ``b *= ratio`` (device decision). Returns
    (kkt, nonfinite_flag)."""
    host = (ctypes.c_double * 2)()
    nat.call("alto_apr_update", nat.ptr(b), b.stride(0), nat.ptr(ratio), ratio.stride(0), b.shape[0],
             rank, tau, apply, host, nat.stream_ptr())
    return float(host[0]), host[1] != 0.0


def loglik_data_term_dview(alto: AltoTensor, dfac: DeviceFactors, weights_dev, partials=None,
                           scaled=None, mode: int = 0):
    """Data term over the decoded view of ``mode`` (the Phi kernel's B-row
    machinery with B = lambda o A_mode); returns a device scalar, no sync."""
    t = nat.torch()
    R = dfac.rank
    _fm, rows, crd, vvals, _recur = device_dview(alto, mode, R)
    if partials is None:
        n = ctypes.c_int32(0)
        nat.call("alto_loglik_dview_partials", alto.nnz, R, ctypes.byref(n))
        partials = t.empty(n.value, dtype=t.float64, device=nat.device())
    a = dfac.mats[mode]
    if scaled is None:
        scaled = t.zeros_like(a)
    scaled[:, :R] = a[:, :R] * weights_dev
    nat.call("alto_loglik_dview", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(rows), nat.ptr(crd),
             nat.ptr(vvals), alto.nnz, ctypes.byref(dfac.struct), mode, nat.ptr(scaled), scaled.stride(0),
             nat.ptr(partials), nat.stream_ptr())
    return partials[-1]


def loglik_data_term_pstream(alto: AltoTensor, dfac: DeviceFactors, weights_dev, mode: int, pi_il,
                             partials=None, scaled=None):
    """Data term from the streamed Khatri-Rao rows of ``mode`` (``pi_il`` as
    stored by that mode's gathering Phi with the current factors of the
    other modes): sum_x v_x log(<lambda o A_mode[row_x], Pi[x]>). Returns a
    device scalar, no sync."""
    t = nat.torch()
    R = dfac.rank
    if partials is None:
        n = ctypes.c_int32(0)
        nat.call("alto_loglik_pstream_partials", ctypes.byref(n))
        partials = t.empty(n.value, dtype=t.float64, device=nat.device())
    a = dfac.mats[mode]
    if scaled is None:
        scaled = t.zeros_like(a)
    scaled[:, :R] = a[:, :R] * weights_dev
    il_rows, il_vals, compact = pstream_view(alto, mode, R)
    nat.call("alto_loglik_pstream2", nat.ptr(il_rows), nat.ptr(il_vals), int(compact), nat.ptr(pi_il), alto.nnz, R,
             nat.ptr(scaled), scaled.stride(0), nat.ptr(partials), partials.numel(), nat.stream_ptr())
    return partials[0]


def loglik_data_term(alto: AltoTensor, dfac: DeviceFactors, weights_dev) -> float:
    t = nat.torch()
    n = ctypes.c_int32(0)
    nat.call("alto_loglik_partials", alto.nnz, ctypes.byref(n))
    partials = t.empty(n.value, dtype=t.float64, device=nat.device())
    out = ctypes.c_double(0.0)
    nat.call("alto_loglik", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(alto._keys),
             nat.ptr(alto._vals), alto.nnz, ctypes.byref(dfac.struct), nat.ptr(weights_dev),
             nat.ptr(partials), ctypes.byref(out), nat.stream_ptr())
    return out.value


def _total_mass(mats, rank: int, weights_dev) -> float:
    prod = None
    for m in mats:
        s = m[:, :rank].sum(dim=0)
        prod = s if prod is None else prod * s
    return float(prod @ weights_dev)


def model_values_at_dev(alto: AltoTensor, model: KruskalModel):
    """Model values at every nonzero (device), for the direct-fit path."""
    t = nat.torch()
    coords = alto.device_coords()
    prod = t.ones((alto.nnz, model.rank), dtype=t.float64, device=coords.device)
    for n, f in enumerate(model.factors):
        prod *= t.from_numpy(f).to(coords.device)[coords[:, n]]
    return prod @ t.from_numpy(model.weights).to(coords.device)


# ---------------------------------------------------------------------------
# public API


def precompute_krp_rows(alto: AltoTensor, factors, mode: int):
    factors = check_factors(factors, alto.shape)
    check_mode(mode, alto.ndim)
    R = factors[0].shape[1]
    pi = launch_pi(alto, DeviceFactors(factors, R), mode)[:, :R]
    return pi if _returns_torch(factors) else pi.cpu().numpy().copy()


def phi_kernel(alto: AltoTensor, scaled, factors, mode: int, *, krp_rows=None, eps: float = 1e-10,
               workers: int = 1, num_segments: int | None = None, strategy="auto",
               temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES, exact=None):
    t = nat.torch()
    factors = check_factors(factors, alto.shape)
    check_mode(mode, alto.ndim)
    rank = factors[0].shape[1]
    sshape = tuple(scaled.shape)
    if sshape != (alto.shape.dims[mode], rank):
        raise ValueError(f"scaled matrix must be {(alto.shape.dims[mode], rank)}, got {sshape}")
    if krp_rows is not None and tuple(krp_rows.shape) != (alto.nnz, rank):
        raise ValueError("krp_rows must be (nnz, rank) in tensor entry order")
    num_segments = num_segments if num_segments is not None else max(workers, 1)
    choice = resolve_strategy(alto, mode, workers, rank, num_segments, strategy, temp_budget_bytes)
    kernel = kernel_for(choice, resolve_exact(exact))
    dfac = DeviceFactors(factors, rank)
    dscaled = nat.to_device_matrix(scaled)
    pi = pi_view = None
    if krp_rows is not None:
        pi = nat.to_device_matrix(krp_rows)
        if kernel == "dview":
            pi_view = pi.index_select(0, dview_order(alto, mode, rank)[0])
        elif kernel in ("exact-output", "oriented"):
            perm = device_mode_view(alto, mode)[0]
            pi_view = pi.index_select(0, perm)
    out = launch_phi(alto, dfac, mode, kernel, dscaled, eps, pi=pi, pi_view=pi_view,
                     num_segments=num_segments)
    res = out[:, :rank]
    as_torch = _returns_torch(factors) or isinstance(scaled, t.Tensor)
    return res if as_torch else res.cpu().numpy().copy()


def kkt_violation(scaled, ratio) -> float:
    return float(np.abs(np.minimum(scaled, 1.0 - ratio)).max())


def select_krp_memory_mode(stats: TensorStats, rank: int,
                           fast_memory_bytes: int = DEFAULT_FAST_MEMORY_BYTES) -> str:
    factor_bytes = sum(stats.shape.dims) * rank * 8
    limited = min(stats.fiber_reuse) < _LOW_REUSE_BELOW
    return "pre" if (limited and factor_bytes > fast_memory_bytes) else "otf"


def poisson_loglik(alto: AltoTensor, model: KruskalModel) -> float:
    t = nat.torch()
    R = model.rank
    dfac = DeviceFactors(model.factors, R)
    w = t.from_numpy(model.weights).to(nat.device())
    total = float(np.prod([f.sum(axis=0) for f in model.factors], axis=0) @ model.weights)
    return loglik_data_term(alto, dfac, w) - total


class AprState:
    """Device state of one CP-APR run; ``outer()`` is one outer iteration
    (the bench's step)."""

    def __init__(self, alto: AltoTensor, config: CpAprConfig, init: KruskalModel | None = None,
                 exact=None, reduce=None):
        """``reduce``: optional in-place cross-rank sum (multi-GPU: ``alto``
        is this rank's ALTO-ordered shard; Phi partials and the
        log-likelihood data term are summed over ranks)."""
        t = nat.torch()
        self.reduce = reduce
        check_nonnegative_values(alto._vals)
        if not bool((t.remainder(alto._vals, 1.0) == 0.0).all()):
            warnings.warn("tensor has non-integer values; the Poisson model assumes counts",
                          stacklevel=3)
        if init is None:
            model = init_factors(alto.shape, config.rank, config.seed, nonneg=True)
        else:
            if init.shape != alto.shape.dims or init.rank != config.rank:
                raise ValueError("initial model does not match the tensor and rank")
            if (init.weights < 0).any() or any((f < 0).any() for f in init.factors):
                raise ValueError("initial model must be nonnegative")
            model = init.copy()
        model = model.normalized(ord=1)
        self.alto = alto
        self.config = config
        R = self.rank = config.rank
        dev = nat.device()
        self.dfac = DeviceFactors(model.factors, R)
        self.weights = t.from_numpy(model.weights.copy()).to(dev)
        stats = compute_stats(alto)
        mm = config.memory_mode
        if mm == "auto":
            mm = select_krp_memory_mode(stats, R, config.fast_memory_bytes)
        self.memory_mode = mm
        nseg = config.num_segments if config.num_segments is not None else max(config.workers, 1)
        self.num_segments = nseg
        self.choices = [
            resolve_strategy(alto, n, config.workers, R, nseg, config.strategy,
                             config.temp_budget_bytes)
            for n in range(alto.ndim)
        ]
        self.exact = resolve_exact(exact)
        self.kernels = [kernel_for(c, self.exact) for c in self.choices]
        if reduce is not None:
            self.kernels = agree_kernels(self.kernels)
        if not nat.env_flag("ALTO_B200_APR_BLOCK", False):
            for n, k in enumerate(self.kernels):
                if k == "dview":
                    prefer_unblocked(alto, n)
        self.ratio_prev = [None] * alto.ndim
        ld = nat.padded_ld(R)
        self.b = [t.zeros((d, ld), dtype=t.float64, device=dev) for d in alto.shape.dims]
        self.kkt_trace, self.inner_counts, self.loglik_trace = [], [], []
        self.inner_loglik = [] if config.track_inner_loglik else None
        self.n_outer = 0
        self.converged = False

    def _pi(self, n: int):
        kernel = self.kernels[n]
        if kernel == "dview":
            return None, launch_pi_dview(self.alto, self.dfac, n)
        if kernel in ("exact-output", "oriented"):
            vkeys = device_mode_view(self.alto, n)[1]
            return None, launch_pi(self.alto, self.dfac, n, keys=vkeys)
        return launch_pi(self.alto, self.dfac, n), None

    def update_mode(self, n: int, outer: int):
        t = nat.torch()
        cfg = self.config
        R = self.rank
        a = self.dfac.mats[n][:, :R]
        b = self.b[n]
        if outer > 1:
            shift = (a < cfg.kappa_tol) & (self.ratio_prev[n][:, :R] > 1.0)
            b[:, :R] = (a + cfg.kappa * shift.to(t.float64)) * self.weights
        else:
            b[:, :R] = a * self.weights
        pi = pi_view = None
        if self.memory_mode == "pre":
            pi, pi_view = self._pi(n)
        ll_inner = []
        track_rows = other_mass = None
        if cfg.track_inner_loglik:
            track_rows = (pi if pi is not None else launch_pi(self.alto, self.dfac, n))[:, :R]
            other_mass = _other_mode_mass(self.dfac.mats, n, R)
            ll_inner.append(_working_loglik(self.alto, b[:, :R], track_rows, n, other_mass))
        if self._device_loop(n):
            return self._inner_device(n, outer, b, pi_view)
        inner_used = 0
        kkt = float("inf")
        all_conv = True
        ratio = None
        for _ in range(cfg.max_inner):
            ratio = launch_phi(self.alto, self.dfac, n, self.kernels[n], b, cfg.eps, pi=pi,
                               pi_view=pi_view, num_segments=self.num_segments)
            if self.reduce is not None:
                self.reduce(ratio)
            inner_used += 1
            kkt, nonfinite = apr_update(b, ratio, R, cfg.tau, apply=-1)
            if kkt < cfg.tau:
                break
            all_conv = False
            if nonfinite:
                raise NumericalError(
                    f"non-finite factor update at outer {outer}, mode {n}, inner {inner_used}")
            if cfg.track_inner_loglik:
                ll_inner.append(_working_loglik(self.alto, b[:, :R], track_rows, n, other_mass))
        self.ratio_prev[n] = ratio
        self._finish_mode(n, b)
        return kkt, inner_used, all_conv, ll_inner

    def _finish_mode(self, n: int, b) -> None:
        t = nat.torch()
        bb = b[:, : self.rank]
        w = bb.sum(dim=0)
        if getattr(self, "_wbuf", None) is not None:
            # graph path: lambda lives in one persistent buffer so a captured
            # outer iteration reads the values of the previous replay
            self._wbuf.copy_(w)
            w = self.weights = self._wbuf
        else:
            self.weights = w
        safe = t.where(w > 0, w, t.ones_like(w))
        self.dfac.mats[n][:, : self.rank] = t.where(w > 0, bb / safe, t.zeros_like(bb))

    def _device_loop(self, n: int) -> bool:
        """The inner loop runs device-driven (one host sync per mode) when
        nothing needs the host between iterations: the dview Phi kernel and
        no per-iteration log-likelihood tracking. Across ranks the Phi
        partials are summed after every launch (stream-ordered collective),
        so every rank takes the same device-side decisions."""
        return (self.kernels[n] == "dview" and not self.config.track_inner_loglik
                and 1 <= self.config.max_inner <= 1024 and not nat.env_flag("ALTO_B200_HOST_INNER"))

    def _pstream_buf(self, n: int):
        """Pi buffer of the streamed-Pi inner iterations, or None when mode
        ``n`` keeps gathering (ALTO_B200_PSTREAM=0, rank > 16, a single
        inner iteration, a non-dview kernel, or not enough free memory for
        Pi plus the slot-ordered views)."""
        if not hasattr(self, "_pil_ok"):
            t = nat.torch()
            R, cfg = self.rank, self.config
            ok = (nat.env_flag("ALTO_B200_PSTREAM", True) and R <= 16 and cfg.max_inner >= 2
                  and self.memory_mode != "pre" and self.alto.nnz > 0)
            if ok:
                slots, pid = pstream_sizes(self.alto, R)
                views = sum(12 * slots for n_ in range(self.alto.ndim) if ("pstream", n_) not in self.alto._cache)
                try:
                    free = t.cuda.mem_get_info()[0]
                except Exception:
                    free = 0
                ok = 8 * pid + views <= 0.6 * free
            self._pil_ok = ok
            self._pil = t.empty(pstream_sizes(self.alto, R)[1], dtype=t.float64, device=nat.device()) if ok else None
        return self._pil if self.kernels[n] == "dview" else None

    def _phi_inner(self, n: int, it: int, b, out, state, pi_view=None, zero: bool = True):
        """Phi of inner iteration ``it`` in a device-driven loop: the first
        one gathers (and stores Pi when streaming), later ones stream Pi."""
        cfg = self.config
        pil = self._pstream_buf(n) if pi_view is None else None
        if pil is not None and it > 0:
            launch_phi_pstream(self.alto, n, self.rank, b, cfg.eps, pil, out, skip=state, zero=zero)
        else:
            launch_phi(self.alto, self.dfac, n, "dview", b, cfg.eps, pi_view=pi_view, out=out, skip=state,
                       zero=zero, pi_il_out=pil)
            # the buffer now holds Pi of mode n; valid for the log-likelihood
            # while the other modes' factors stay as they are
            self._pil_mode = n if pil is not None else None

    def _ll_stream_mode(self):
        """The mode whose stored Pi can serve the log-likelihood (the last
        mode of the outer iteration: every other factor is final), or None."""
        last = self.alto.ndim - 1
        if getattr(self, "_pil_mode", None) == last and nat.env_flag("ALTO_B200_PSTREAM_LL", True):
            return last
        return None

    def _ll_data_stream(self, mode: int):
        t = nat.torch()
        if getattr(self, "_ll_ps_partials", None) is None:
            n = ctypes.c_int32(0)
            nat.call("alto_loglik_pstream_partials", ctypes.byref(n))
            self._ll_ps_partials = t.empty(n.value, dtype=t.float64, device=nat.device())
            self._ll_ps_scaled = t.zeros_like(self.dfac.mats[mode])
        return loglik_data_term_pstream(self.alto, self.dfac, self.weights, mode, self._pil,
                                        self._ll_ps_partials, self._ll_ps_scaled)

    def _inner_iterations(self, n: int, b, ratio, state, pi_view=None) -> None:
        """Queue mode n's max_inner device-driven iterations (no host read):
        each a no-op once the state says the loop is done."""
        cfg = self.config
        st = nat.stream_ptr()
        if self.reduce is None:
            for it in range(cfg.max_inner):
                self._phi_inner(n, it, b, ratio, state, pi_view)
                nat.call("alto_apr_inner_step", nat.ptr(b), b.stride(0), nat.ptr(ratio), ratio.stride(0),
                         b.shape[0], self.rank, cfg.tau, it, nat.ptr(state), st)
            return
        # the collective runs every iteration on every rank: the partial
        # buffer is zeroed unconditionally (a skipped Phi contributes 0)
        # and the last executed iteration's reduced Phi is kept aside.
        # The copy precedes the step: `done` then reflects only earlier
        # iterations, so the iteration that converges (kkt < tau) still
        # lands in `ratio` (the next outer's shift reads it, apr.py:270).
        # One partial buffer per mode, allocated before any graph capture.
        parts = getattr(self, "_parts", None)
        if parts is None:
            parts = self._parts = [None] * self.alto.ndim
        part = parts[n]
        if part is None or part.shape != ratio.shape:
            part = parts[n] = nat.torch().empty_like(ratio)
        for it in range(cfg.max_inner):
            part.zero_()
            self._phi_inner(n, it, b, part, state, pi_view, zero=False)
            self.reduce(part)
            nat.call("alto_copy_if", nat.ptr(part), nat.ptr(ratio), part.numel(), nat.ptr(state), st)
            nat.call("alto_apr_inner_step", nat.ptr(b), b.stride(0), nat.ptr(part), part.stride(0),
                     b.shape[0], self.rank, cfg.tau, it, nat.ptr(state), st)

    def _reduce_capturable(self) -> bool:
        """A cross-rank sum that may sit inside a CUDA graph: the library's
        own NCCL communicator (distributed.NativeComm: a C call on the current
        stream); ALTO_B200_DIST_GRAPH=0 keeps multi-rank outers eager."""
        from ..distributed import NativeComm

        return (isinstance(getattr(self.reduce, "__self__", None), NativeComm)
                and nat.env_flag("ALTO_B200_DIST_GRAPH", True))

    def _inner_device(self, n: int, outer: int, b, pi_view):
        t = nat.torch()
        cfg = self.config
        if getattr(self, "_inner_state", None) is None:
            size = ctypes.c_size_t(0)
            nat.call("alto_apr_inner_state_bytes", cfg.max_inner, ctypes.byref(size))
            self._inner_state = t.empty(size.value, dtype=t.uint8, device=nat.device())
            self._ratio = [None] * self.alto.ndim
        if self._ratio[n] is None:
            # zeroed: with a cross-rank reduction the kept Phi is copied in
            # conditionally, and the next outer's shift reads it
            self._ratio[n] = t.zeros((self.alto.shape.dims[n], nat.padded_ld(self.rank)), dtype=t.float64,
                                     device=nat.device())
        state, ratio, st = self._inner_state, self._ratio[n], nat.stream_ptr()
        nat.call("alto_apr_inner_reset", nat.ptr(state), st)
        self._inner_iterations(n, b, ratio, state, pi_view)
        used, bad, kkt = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_double(0.0)
        nat.call("alto_apr_inner_result", nat.ptr(state), ctypes.byref(used), ctypes.byref(bad),
                 ctypes.byref(kkt), st)
        if bad.value:
            raise NumericalError(f"non-finite factor update at outer {outer}, mode {n}, inner {bad.value}")
        # converged in this mode iff the very first iteration broke out
        all_conv = used.value == 1 and kkt.value < cfg.tau
        # the ratio buffer is reused per mode: keep a copy for next outer's shift
        self.ratio_prev[n] = ratio.clone()
        self._finish_mode(n, b)
        return kkt.value, used.value, all_conv, []

    # ---- device-resident outer iteration (CUDA graph) ----------------------

    def _graph_ok(self) -> bool:
        return (self.memory_mode != "pre" and (self.reduce is None or self._reduce_capturable())
                and all(self._device_loop(n) for n in range(self.alto.ndim))
                and not nat.env_flag("ALTO_B200_NO_GRAPH"))

    def _setup_graph_state(self):
        t = nat.torch()
        cfg = self.config
        dev = nat.device()
        N = self.alto.ndim
        size = ctypes.c_size_t(0)
        nat.call("alto_apr_inner_state_bytes", cfg.max_inner, ctypes.byref(size))
        off = ctypes.c_size_t(0)
        nat.call("alto_apr_inner_kkt_offset", ctypes.byref(off))
        self._kkt_off = off.value
        self._states = [t.zeros(size.value, dtype=t.uint8, device=dev) for _ in range(N)]
        self._ratio = [t.zeros((d, nat.padded_ld(self.rank)), dtype=t.float64, device=dev)
                       for d in self.alto.shape.dims]
        nb = self._kkt_off + 8 * cfg.max_inner
        self._hstates = [t.empty(nb, dtype=t.uint8, pin_memory=True) for _ in range(N)]
        n = ctypes.c_int32(0)
        nat.call("alto_loglik_partials", self.alto.nnz, ctypes.byref(n))
        self._ll_partials = t.empty(n.value, dtype=t.float64, device=dev)
        nat.call("alto_loglik_dview_partials", self.alto.nnz, self.rank, ctypes.byref(n))
        self._ll_dv_partials = t.empty(n.value, dtype=t.float64, device=dev)
        self._ll_scaled = t.zeros_like(self.dfac.mats[0])
        self._hll = t.empty(2, dtype=t.float64, pin_memory=True)
        self._wbuf = self.weights.clone()
        self.weights = self._wbuf
        self._graph = None

    def _outer_device_body(self, shift: bool):
        """One outer iteration, stream-ordered with no host round trip:
        per mode the B update, the device-driven inner loop and the
        normalisation; then the log-likelihood. Results land in pinned
        buffers (read after one sync)."""
        t = nat.torch()
        cfg = self.config
        R = self.rank
        st = nat.stream_ptr()
        for n in range(self.alto.ndim):
            a = self.dfac.mats[n][:, :R]
            b = self.b[n]
            if shift:
                sh = (a < cfg.kappa_tol) & (self._ratio[n][:, :R] > 1.0)
                b[:, :R] = (a + cfg.kappa * sh.to(t.float64)) * self.weights
            else:
                b[:, :R] = a * self.weights
            state, ratio = self._states[n], self._ratio[n]
            nat.call("alto_apr_inner_reset", nat.ptr(state), st)
            self._inner_iterations(n, b, ratio, state)
            hs = self._hstates[n]
            hs[:16].copy_(state[:16], non_blocking=True)
            hs[self._kkt_off:].copy_(state[self._kkt_off:self._kkt_off + 8 * cfg.max_inner], non_blocking=True)
            self._finish_mode(n, b)
        ll_mode = self._ll_stream_mode()
        if ll_mode is not None:
            data = self._ll_data_stream(ll_mode)
        elif self.kernels[0] == "dview":
            data = loglik_data_term_dview(self.alto, self.dfac, self.weights, self._ll_dv_partials,
                                          self._ll_scaled)
        else:
            nat.call("alto_loglik", ctypes.byref(nat.layout_struct(self.alto.layout)), nat.ptr(self.alto._keys),
                     nat.ptr(self.alto._vals), self.alto.nnz, ctypes.byref(self.dfac.struct),
                     nat.ptr(self.weights), nat.ptr(self._ll_partials), None, st)
            data = self._ll_partials[-1]
        if self.reduce is not None:
            self.reduce(data)
        mass = None
        for m in self.dfac.mats:
            s = m[:, :R].sum(dim=0)
            mass = s if mass is None else mass * s
        self._hll.copy_(t.stack([data, mass @ self.weights]), non_blocking=True)

    def _outer_graph(self):
        import numpy as _np

        t = nat.torch()
        cfg = self.config
        N = self.alto.ndim
        if not hasattr(self, "_states"):
            self._setup_graph_state()
        shift = self.n_outer > 1
        if shift and self._graph is None and self.n_outer > 2:
            g = t.cuda.CUDAGraph()
            with nat.graph_capture(g):
                self._outer_device_body(True)
            self._graph = g
        if self._graph is not None:
            self._graph.replay()
        else:
            self._outer_device_body(shift)
        done = t.cuda.Event()
        done.record()
        done.synchronize()
        all_conv = True
        kkts, inners = [], []
        for n in range(N):
            hs = self._hstates[n].numpy()
            head = hs[:16].view(_np.int32)
            bad, used = int(head[1]), int(head[2])
            if bad:
                raise NumericalError(f"non-finite factor update at outer {self.n_outer}, mode {n}, inner {bad}")
            kkt = float(hs[self._kkt_off:].view(_np.float64)[used - 1]) if used else float("nan")
            all_conv &= used == 1 and kkt < cfg.tau
            kkts.append(kkt)
            inners.append(used)
            self.ratio_prev[n] = self._ratio[n]
        self.kkt_trace.append(kkts)
        self.inner_counts.append(inners)
        data, mass = (float(x) for x in self._hll.numpy())
        self.loglik_trace.append(data - mass)
        if all_conv:
            self.converged = True
        return all_conv

    def outer(self):
        self.n_outer += 1
        if not getattr(self, "_graph", None):
            self._pil_mode = None  # set again by this outer's gathering Phi
        if self._graph_ok():
            return self._outer_graph()
        all_conv = True
        kkts, inners, lls = [], [], []
        for n in range(self.alto.ndim):
            kkt, used, conv, ll = self.update_mode(n, self.n_outer)
            all_conv &= conv
            kkts.append(kkt)
            inners.append(used)
            lls.append(ll)
        self.kkt_trace.append(kkts)
        self.inner_counts.append(inners)
        if self.inner_loglik is not None:
            self.inner_loglik.append(lls)
        self.loglik_trace.append(self.loglik())
        if all_conv:
            self.converged = True
        return all_conv

    def loglik(self) -> float:
        ll_mode = self._ll_stream_mode()
        if ll_mode is not None:
            data = float(self._ll_data_stream(ll_mode))
        elif self.kernels[0] == "dview":
            data = float(loglik_data_term_dview(self.alto, self.dfac, self.weights))
        else:
            data = loglik_data_term(self.alto, self.dfac, self.weights)
        if self.reduce is not None:
            t = nat.torch()
            d = t.tensor([data], dtype=t.float64, device=self.weights.device)
            self.reduce(d)
            data = float(d.item())
        return data - _total_mass(self.dfac.mats, self.rank, self.weights)

    def model(self) -> KruskalModel:
        R = self.rank
        return KruskalModel(self.weights.cpu().numpy(), [m[:, :R].cpu().numpy() for m in self.dfac.mats])


def cp_apr_mu(alto: AltoTensor, config: CpAprConfig, init: KruskalModel | None = None, *,
              exact=None) -> CpAprResult:
    start = time.perf_counter()
    st = AprState(alto, config, init, exact)
    for _ in range(config.max_outer):
        if st.outer():
            break
    nat.torch().cuda.synchronize()
    return CpAprResult(
        model=st.model(),
        kkt_trace=st.kkt_trace,
        inner_iters=st.inner_counts,
        loglik_trace=st.loglik_trace,
        n_outer=st.n_outer,
        converged=st.converged,
        memory_mode=st.memory_mode,
        strategies=list(st.choices),
        inner_loglik=st.inner_loglik,
        wall_time_s=time.perf_counter() - start,
    )


def _other_mode_mass(mats, mode: int, rank: int):
    mass = None
    for m, f in enumerate(mats):
        if m == mode:
            continue
        s = f[:, :rank].sum(dim=0)
        mass = s if mass is None else mass * s
    if mass is None:
        return nat.torch().ones(rank, dtype=nat.torch().float64, device=mats[0].device)
    return mass


def _working_loglik(alto: AltoTensor, b, krp_rows, mode: int, other_mass) -> float:
    """Log-likelihood of the mid-update model (pkg/src/alto/cpd/apr.py:359-366)."""
    t = nat.torch()
    rows = alto.device_coords()[:, mode]
    mhat = (b[rows] * krp_rows).sum(dim=1)
    logs = t.log(mhat)
    return float(alto._vals @ logs) - float(b.sum(dim=0) @ other_mass)
