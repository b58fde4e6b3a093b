"""CP-ALS with device-resident factors (pkg/src/alto/cpd/als.py:29-158).

Per sweep and mode: hadamard chain of Grams (R x R, host), MTTKRP on the GPU
(the hot path), the normal-equation solve over I_n rows on the device,
column normalisation and the new Gram on the device. Only R-sized vectors and
R x R matrices cross to the host inside the loop.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .. import _native as nat
from ..kernels import (
    DEFAULT_TEMP_BUDGET_BYTES,
    DeviceFactors,
    StrategyChoice,
    _zeros_out,
    kernel_for,
    launch_mttkrp,
    resolve_exact,
    resolve_strategy,
)
from ..tensor import AltoTensor
from ..validation import NumericalError, check_rank, check_workers
from .linalg import gram_dev, hadamard_chain, solve_pseudo_dev
from .model import KruskalModel, init_factors


@dataclass(frozen=True)
class CpAlsConfig:
    rank: int = 16
    max_iters: int = 50
    fit_tol: float = 1e-5
    seed: int = 0
    workers: int = 1
    num_segments: int | None = None
    strategy: str = "auto"
    temp_budget_bytes: int = DEFAULT_TEMP_BUDGET_BYTES

    def __post_init__(self):
        check_rank(self.rank)
        check_workers(self.workers)
        if self.max_iters < 0:
            raise ValueError("max_iters must be >= 0")
        if self.fit_tol <= 0:
            raise ValueError("fit_tol must be positive")


@dataclass
class CpAlsResult:
    model: KruskalModel
    fit_trace: list
    objective_trace: list
    n_iters: int
    converged: bool
    strategies: list = field(default_factory=list)
    wall_time_s: float = 0.0

    @property
    def fit(self) -> float:
        return self.fit_trace[-1]


class AlsState:
    """Device state of one CP-ALS run; ``sweep()`` is one full iteration
    (the bench's step)."""

    def __init__(self, alto: AltoTensor, config: CpAlsConfig, init: KruskalModel | None = None,
                 exact=None, reduce=None, norm_x_sq: float | None = None, row_comm=None, memo=None):
        """``reduce``: optional in-place cross-rank sum applied to every
        MTTKRP output (multi-GPU: ``alto`` is this rank's shard).
        ``row_comm``: a ``distributed.RowComm`` instead -- the partials are
        reduce-scattered to row owners, each rank solves and normalises its
        row block and the blocks are all-gathered (device update path; the
        host path falls back to an all-reduce of the partials)."""
        if init is None:
            model = init_factors(alto.shape, config.rank, config.seed)
        else:
            if init.shape != alto.shape.dims or init.rank != config.rank:
                raise ValueError("initial model does not match the tensor and rank")
            model = init.copy()
        model = model.normalized(ord=2)
        self.alto = alto
        self.config = config
        self.rank = config.rank
        self.weights = model.weights
        self.dfac = DeviceFactors(model.factors, self.rank)
        self.reduce = reduce
        self.row_comm = row_comm
        self.memo = memo  # None: decided by _memo_wanted
        if row_comm is not None and reduce is not None:
            raise ValueError("give either reduce or row_comm")
        self.norm_x_sq = float(alto._vals @ alto._vals) if norm_x_sq is None else norm_x_sq
        self.grams = [gram_dev(m[:, : self.rank]) for m in self.dfac.mats]
        nseg = config.num_segments if config.num_segments is not None else max(config.workers, 1)
        self.num_segments = nseg
        self.exact = resolve_exact(exact)
        self.choices: list[StrategyChoice] = [
            resolve_strategy(alto, n, config.workers, self.rank, nseg, config.strategy,
                             config.temp_budget_bytes)
            for n in range(alto.ndim)
        ]
        self.kernels = [kernel_for(c, self.exact) for c in self.choices]
        self.outs = [None] * alto.ndim
        self.last_mt = None

    def _memo(self):
        """Memoised-sweep plans (``memo.MemoPlan``) for the cyclic mode pairs
        (0, 1), (1, 2), (2, 0) of a 3-mode tensor on the fast decoded-view
        kernels, or None (``ALTO_B200_MEMO=0`` disables them). Returns the
        plan of pair (0, 1) (the bench reports it); ``self._memo_plans``
        holds all three."""
        if not hasattr(self, "_memo_plans"):
            self._memo_plans = None
            alto = self.alto
            if (alto.ndim == 3 and not self.exact and alto.nnz > 0 and self.kernels == ["dview"] * 3
                    and self._memo_wanted()):
                import torch

                from ..memo import MemoPlan
                try:
                    free = torch.cuda.mem_get_info()[0]
                except Exception:
                    free = 0
                if 3 * MemoPlan.bytes_needed(alto, self.rank) <= 0.6 * free:
                    self._memo_plans = {(n, (n + 1) % 3): MemoPlan(alto, self.rank, n, (n + 1) % 3)
                                        for n in range(3)}
        return None if self._memo_plans is None else self._memo_plans[(0, 1)]

    # a memoised sweep saves ~0.6 ms on c2 (2.2 vs 2.85 ms) and its layouts
    # cost ~10 ms more to build than the plain path's: below this many
    # iterations a cold run is faster without them (bench drivers_e2e)
    MEMO_MIN_ITERS = 16

    def _memo_wanted(self) -> bool:
        """ALTO_B200_MEMO=1/0 forces the memoised sweep on/off; otherwise
        (and unless AlsState(memo=...) decided) it runs when the iteration
        budget amortises its build or its layouts are already cached on the
        tensor (a previous memoised run)."""
        env = os.environ.get("ALTO_B200_MEMO")
        if env is not None and env.strip():
            return nat.env_flag("ALTO_B200_MEMO", True)
        if self.memo is not None:
            return bool(self.memo)
        if self.config.max_iters >= self.MEMO_MIN_ITERS:
            return True
        return any(isinstance(k, tuple) and k and k[0] == "memo_cons" for k in self.alto._cache)

    def _memo_state(self):
        return None if not self._memo_plans else tuple(p.t_valid for p in self._memo_plans.values())

    def _set_memo_state(self, state) -> None:
        if self._memo_plans and state is not None:
            for p, v in zip(self._memo_plans.values(), state):
                p.t_valid = v

    def mttkrp(self, n: int):
        """MTTKRP of mode n. Memoised sweep: consume the partial sums the
        previous mode stored for this one when they are valid (one gathered
        row per piece), else produce: this mode's MTTKRP plus the partial
        sums for the next mode. Updating mode n afterwards invalidates the
        sums over mode n (pair (n+1, n+2)). Over two sweeps the pattern is
        produce/consume/produce, consume/produce/consume."""
        if self._memo() is not None:
            plans = self._memo_plans
            prev, nxt = (n - 1) % 3, (n + 1) % 3
            if self.outs[n] is None:
                self.outs[n] = _zeros_out(self.alto.shape.dims[n], self.rank)
            cons = plans[(prev, n)]
            if cons.t_valid:
                cons.mttkrp_m1(self.dfac, self.outs[n])
                cons.t_valid = False
            else:
                plans[(n, nxt)].mttkrp_m0(self.alto, self.dfac, self.outs[n])
            plans[(nxt, (n + 2) % 3)].t_valid = False  # its sums run over mode n
            if self.reduce is not None:
                self.reduce(self.outs[n])
            return self.outs[n][:, : self.rank]
        self.outs[n] = launch_mttkrp(self.alto, self.dfac, n, self.kernels[n],
                                     num_segments=self.num_segments, out=self.outs[n])
        if self.reduce is not None:
            self.reduce(self.outs[n])
        return self.outs[n][:, : self.rank]

    def update_mode(self, n: int):
        import torch

        R = self.rank
        v = hadamard_chain(self.grams, skip=n)
        mt = self.mttkrp(n)
        a = solve_pseudo_dev(mt, v)
        norms = torch.linalg.vector_norm(a, dim=0)
        safe = torch.where(norms == 0.0, torch.ones_like(norms), norms)
        a = a / safe
        self.weights = norms.cpu().numpy()
        self.dfac.mats[n][:, :R].copy_(a)
        self.grams[n] = gram_dev(self.dfac.mats[n][:, :R])
        self.last_mt = mt

    # ---- device-resident sweep (solve, normalisation and Grams on the GPU) ----

    def _device_ok(self) -> bool:
        return (not self.exact and self.rank <= 32 and self.alto.ndim >= 2
                and not nat.env_flag("ALTO_B200_HOST_ALS"))

    def _setup_device(self):
        import ctypes

        import torch

        t, dev = torch, nat.device()
        N, R = self.alto.ndim, self.rank
        ld = nat.padded_ld(R)
        self._dgrams = t.from_numpy(np.stack([np.asarray(g, dtype=np.float64) for g in self.grams])).to(dev)
        self._dweights = t.zeros(R, dtype=t.float64, device=dev)
        self._dflags = t.zeros(2, dtype=t.int32, device=dev)
        self._hflags = t.zeros(2, dtype=t.int32, pin_memory=True)
        self._hgrams = t.empty((N, R, R), dtype=t.float64, pin_memory=True)
        if not hasattr(self, "_norms_host"):
            self._norms_host = t.empty(R, dtype=t.float64, pin_memory=True)
        need = 0
        for n in range(N):
            b = ctypes.c_size_t(0)
            nat.call("alto_als_update_scratch_bytes", self.alto.shape.dims[n], R, ctypes.byref(b))
            need = max(need, b.value)
        self._als_scratch = t.empty(need, dtype=t.uint8, device=dev)
        rc = self.row_comm
        if rc is not None:
            # factors and MTTKRP outputs padded to W * chunk rows (the
            # collectives need equal blocks); the factor the kernels read is
            # the leading I_n rows of the padded buffer
            self._pads, self._blk_out, self._blk_a = [], [], []
            for n in range(N):
                rows = self.alto.shape.dims[n]
                pad = t.zeros((rc.padded(rows), ld), dtype=t.float64, device=dev)
                pad[:rows].copy_(self.dfac.mats[n])
                self.dfac.mats[n] = pad[:rows]
                self._pads.append(pad)
                self.outs[n] = t.zeros((rc.padded(rows), ld), dtype=t.float64, device=dev)
                self._blk_out.append(t.zeros((rc.chunk(rows), ld), dtype=t.float64, device=dev))
                self._blk_a.append(t.zeros((rc.chunk(rows), ld), dtype=t.float64, device=dev))
                b = ctypes.c_size_t(0)
                nat.call("alto_als_update_scratch_bytes", rc.chunk(rows), R, ctypes.byref(b))
                need = max(need, b.value)
            self._als_scratch = t.empty(need, dtype=t.uint8, device=dev)
            self.dfac.struct = nat.factors_struct(self.dfac.mats, R)
            self._gram_raw = t.zeros(R * R, dtype=t.float64, device=dev)
        for n in range(N):
            if self.outs[n] is None:
                self.outs[n] = t.zeros((self.alto.shape.dims[n], ld), dtype=t.float64, device=dev)
        self._snap = [m.clone() for m in self.dfac.mats]
        self._snap_grams = self._dgrams.clone()
        self._graph = None
        self._graphs = {}
        self._eager_sweeps = 0
        self._side_stream = t.cuda.Stream()

    def _sweep_device_body(self):
        """Everything of one sweep, stream-ordered, no host round trip
        (capturable in a CUDA graph)."""
        import ctypes

        N, R = self.alto.ndim, self.rank
        for n in range(N):
            self._snap[n].copy_(self.dfac.mats[n])
        self._snap_grams.copy_(self._dgrams)
        self._dflags.zero_()
        import torch

        main = torch.cuda.current_stream()
        st = nat.stream_ptr()
        side = self._side_stream
        for n in range(N):
            # the Cholesky factor of mode n's normal matrix needs only the
            # Gram matrices (final after mode n-1's update): it runs on a
            # side stream while mode n's MTTKRP runs (fork/join, also inside
            # the captured graph)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                nat.call("alto_als_chol", nat.ptr(self._dgrams), N, n, R, nat.ptr(self._als_scratch),
                         self._als_scratch.numel(), nat.ptr(self._dflags), nat.stream_ptr())
            self.mttkrp(n)
            main.wait_stream(side)
            out, mat = self.outs[n], self.dfac.mats[n]
            if self.row_comm is not None:
                self._row_owner_update(n, st)
                continue
            nat.call("alto_als_update_solve", nat.ptr(out), out.stride(0), self.alto.shape.dims[n], R,
                     nat.ptr(self._dgrams), N, n, nat.ptr(mat), mat.stride(0), nat.ptr(self._dweights),
                     nat.ptr(self._als_scratch), self._als_scratch.numel(), nat.ptr(self._dflags), 0, st)
        if self.row_comm is not None:
            # a failed solve on any rank takes every rank to the same fallback
            self.row_comm.all_reduce_max(self._dflags)
        self._hflags.copy_(self._dflags, non_blocking=True)
        self._hgrams.copy_(self._dgrams, non_blocking=True)
        self._norms_host.copy_(self._dweights, non_blocking=True)

    def _row_owner_update(self, n: int, st) -> None:
        """Mode n's update with row owners: reduce-scatter the partial, solve
        this rank's rows, all-reduce the raw Gram, normalise, all-gather."""
        N, R, rc = self.alto.ndim, self.rank, self.row_comm
        out, blk, a = self.outs[n], self._blk_out[n], self._blk_a[n]
        rc.reduce_scatter(blk, out)
        nat.call("alto_als_solve_gram", nat.ptr(blk), blk.stride(0), blk.shape[0], R, nat.ptr(self._dgrams), N, n,
                 nat.ptr(a), a.stride(0), nat.ptr(self._als_scratch), self._als_scratch.numel(),
                 nat.ptr(self._dflags), 0, nat.ptr(self._gram_raw), st)
        rc.all_reduce(self._gram_raw)
        nat.call("alto_als_normalize", nat.ptr(self._gram_raw), R, nat.ptr(self._dgrams), N, n, nat.ptr(a),
                 a.stride(0), a.shape[0], nat.ptr(self._dweights), nat.ptr(self._als_scratch),
                 self._als_scratch.numel(), st)
        rc.all_gather(self._pads[n], a)

    def _graph_capturable(self) -> bool:
        """Collectives inside the sweep graph: the library's own NCCL
        communicator (distributed.NativeComm, a C call on the current stream)
        by default (ALTO_B200_DIST_GRAPH=0 keeps it eager); torch.distributed
        NCCL only with ALTO_B200_DIST_GRAPH=1; gloo never (host staging)."""
        from ..distributed import NativeComm

        comm = self.row_comm if self.row_comm is not None else getattr(self.reduce, "__self__", None)
        if isinstance(comm, NativeComm):
            return nat.env_flag("ALTO_B200_DIST_GRAPH", True)
        if self.reduce is not None:
            return False
        if self.row_comm is not None:
            return not self.row_comm.gloo and nat.env_flag("ALTO_B200_DIST_GRAPH", False)
        return True

    def _sweep_device(self):
        import torch

        N, R = self.alto.ndim, self.rank
        use_graph = self._graph_capturable() and not nat.env_flag("ALTO_B200_NO_GRAPH")
        # one graph per memo state at the sweep's start (the memoised sweep
        # alternates between two kernel sequences); the Python-side memo
        # flags are set to the state the captured sequence leaves behind
        self._memo()
        start = self._memo_state()
        self._sweep_start_state = start
        graph = self._graphs.get(start)
        if graph is None and use_graph and self._eager_sweeps >= 1:
            g = torch.cuda.CUDAGraph()
            with nat.graph_capture(g):
                self._sweep_device_body()
            graph = self._graphs[start] = (g, self._memo_state())
            self._set_memo_state(start)
        if graph is not None:
            graph[0].replay()
            self._set_memo_state(graph[1])
            self._graph = graph[0]
        else:
            self._sweep_device_body()
            self._eager_sweeps += 1
        done = torch.cuda.Event()
        done.record()
        done.synchronize()
        flags = self._hflags.numpy()
        if flags[0]:
            raise ValueError("non-finite input to the normal-equation solve")
        if flags[1]:
            # not positive definite: restore the sweep's start and take the
            # host path (eigh pseudo-inverse, pkg/src/alto/cpd/linalg.py:47-52)
            for n in range(N):
                self.dfac.mats[n].copy_(self._snap[n])
            self._dgrams.copy_(self._snap_grams)
            self._set_memo_state(self._sweep_start_state)
            self.grams = [g.copy() for g in self._dgrams.cpu().numpy()]
            self._sweep_host()
            self._dgrams.copy_(torch.from_numpy(np.stack(self.grams)))
            return
        self.grams = [g.copy() for g in self._hgrams.numpy()]
        self._norms_ready = done
        self._weights = None
        if self.row_comm is not None:
            self.last_mt = self._blk_out[N - 1][:, :R]
            self._last_a = self._blk_a[N - 1][:, :R]
        else:
            self.last_mt = self.outs[N - 1][:, :R]
            self._last_a = None

    def sweep(self):
        """One CP-ALS iteration. Device path (fast kernels, R <= 32): the
        normal equations, normalisation and Grams run on the GPU and the
        whole sweep replays as one CUDA graph, one host sync per sweep."""
        if self._device_ok():
            if not hasattr(self, "_dgrams"):
                self._setup_device()
            return self._sweep_device()
        return self._sweep_host()

    def _sweep_host(self):
        """One CP-ALS iteration, pipelined: the MTTKRP of mode n+1 only needs
        the updated factor n, so it is enqueued before the host waits for
        mode n's Gram (R x R, needed for mode n+1's normal equations); the
        host-side factorisation overlaps the next kernel. Non-finite input
        to the solve is reported at the end of the sweep."""
        import torch

        R = self.rank
        N = self.alto.ndim
        if self.row_comm is not None:
            # host path with row owners: every rank takes the full summed
            # partial (all-reduce) and updates every row
            self.reduce = self.row_comm.all_reduce
            self._last_a = None
            try:
                return self._sweep_host_body(R, N)
            finally:
                self.reduce = None
        self._last_a = None
        return self._sweep_host_body(R, N)

    def _sweep_host_body(self, R: int, N: int):
        import torch

        if not hasattr(self, "_gram_host"):
            self._gram_host = [torch.empty((R, R), dtype=torch.float64, pin_memory=True) for _ in range(N)]
        mt = self.mttkrp(0)
        norms = None
        for n in range(N):
            v = hadamard_chain(self.grams, skip=n)
            a = solve_pseudo_dev(mt, v, check_finite=False)
            norms = torch.linalg.vector_norm(a, dim=0)
            safe = torch.where(norms == 0.0, torch.ones_like(norms), norms)
            mat = self.dfac.mats[n][:, :R]
            mat.copy_(a / safe)
            self._gram_host[n].copy_(mat.T @ mat, non_blocking=True)
            done = torch.cuda.Event()
            done.record()
            self.last_mt = mt
            if n + 1 < N:
                mt = self.mttkrp(n + 1)
            done.synchronize()
            self.grams[n] = self._gram_host[n].numpy().copy()
            if not np.isfinite(self.grams[n]).all():
                raise ValueError("non-finite input to the normal-equation solve")
        # lambda read back lazily (pinned copy + event): no sync per sweep
        if not hasattr(self, "_norms_host"):
            self._norms_host = torch.empty(R, dtype=torch.float64, pin_memory=True)
        self._norms_host.copy_(norms, non_blocking=True)
        self._norms_ready = torch.cuda.Event()
        self._norms_ready.record()
        self._weights = None

    @property
    def weights(self) -> np.ndarray:
        if self._weights is None:
            self._norms_ready.synchronize()
            self._weights = self._norms_host.numpy().copy()
        return self._weights

    @weights.setter
    def weights(self, value) -> None:
        self._weights = value

    def fit(self):
        import torch

        N = self.alto.ndim
        R = self.rank
        w = torch.from_numpy(self.weights).to(self.last_mt.device)
        if getattr(self, "_last_a", None) is not None:
            # row owners: this rank's rows of <M_N, A_N diag(w)>, summed over ranks
            part = (self.last_mt * self._last_a * w).sum().reshape(1)
            inner = float(self.row_comm.all_reduce(part).item())
        else:
            inner = float((self.last_mt * self.dfac.mats[N - 1][:, :R] * w).sum())
        model_norm_sq = float(self.weights @ (hadamard_chain(self.grams) @ self.weights))
        res_sq = max(self.norm_x_sq - 2.0 * inner + model_norm_sq, 0.0)
        return 1.0 - math.sqrt(res_sq / self.norm_x_sq), res_sq

    def model(self) -> KruskalModel:
        R = self.rank
        return KruskalModel(self.weights.copy(), [m[:, :R].cpu().numpy() for m in self.dfac.mats])


def cp_als(alto: AltoTensor, config: CpAlsConfig, init: KruskalModel | None = None, *,
           exact=None) -> CpAlsResult:
    start = time.perf_counter()
    st = AlsState(alto, config, init, exact)
    if config.max_iters == 0:
        fit, res_sq = _fit_direct(alto, st.model(), st.norm_x_sq)
        return CpAlsResult(st.model(), [fit], [res_sq], 0, False, [],
                           time.perf_counter() - start)
    fit_trace, objective_trace = [], []
    prev_fit = None
    converged = False
    n_iters = 0
    for it in range(1, config.max_iters + 1):
        n_iters = it
        st.sweep()
        fit, res_sq = st.fit()
        if not math.isfinite(fit):
            raise NumericalError(f"fit became non-finite at iteration {it}")
        fit_trace.append(fit)
        objective_trace.append(res_sq)
        if prev_fit is not None and abs(fit - prev_fit) < config.fit_tol:
            converged = True
            break
        prev_fit = fit
    nat.torch().cuda.synchronize()
    return CpAlsResult(st.model(), fit_trace, objective_trace, n_iters, converged,
                       list(st.choices), time.perf_counter() - start)


def _fit_direct(alto: AltoTensor, model: KruskalModel, norm_x_sq: float):
    from .apr import model_values_at_dev

    inner = float(alto._vals @ model_values_at_dev(alto, model))
    res_sq = max(norm_x_sq - 2.0 * inner + model.norm_squared(), 0.0)
    return 1.0 - math.sqrt(res_sq / norm_x_sq), res_sq
