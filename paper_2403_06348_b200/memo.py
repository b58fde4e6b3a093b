"""Memoised CP-ALS sweep for 3-mode tensors (csrc/memo.cu, memo0_kernel in
csrc/dview_kernels.cu).

CP-ALS updates the modes in order (pkg/src/alto/cpd/als.py:84-96). With
modes (m0, m1, k) = (0, 1, 2) the MTTKRPs of m0 and m1 share the partial
sums T[i, j] = sum_k v_ijk A_k[k] (A_k does not change between the two
updates): the m0 pass stores T once per (i, j) piece of its view, the m1 pass
reads T through a position -> piece index and gathers one factor row per
piece instead of two per nonzero.
The reference has no counterpart (it recomputes every MTTKRP); results match
it to rounding (fast path, tests <= 1e-12 relative)."""

from __future__ import annotations

import ctypes
import types

from . import _native as nat
from .tensor import AltoTensor


def _lanes(rank: int) -> int:
    g = 1
    while 4 * g < rank:
        g *= 2
    return g


class MemoPlan:
    """Views, piece index and T buffer of the memoised pair (m0, m1)."""

    def __init__(self, alto: AltoTensor, rank: int, m0: int = 0, m1: int = 1):
        if alto.ndim != 3:
            raise ValueError("the memoised sweep needs a 3-mode tensor")
        t = nat.torch()
        self.m0, self.m1, self.rank = m0, m1, rank
        self.T = None
        self.t_valid = False
        self.k = 3 - m0 - m1
        self.jplane = m1 if m1 < m0 else m1 - 1
        # producer (profiles/r02_fused_producer_ab.txt): the branch-free fused
        # kernel over an interleaved (rows, j | piece start, k, slot, v) stream
        # staged with bulk copies, storing T at the consumer's slots
        # (csrc/memo_sums.cu, rank <= 32); ALTO_B200_MEMO_KERNEL=memo0 keeps
        # the round-2 fused kernel over the plain view (also the path for
        # rank > 32 and deterministic mode)
        kind = nat.env_str("ALTO_B200_MEMO_KERNEL", "fused").lower()
        if kind not in ("fused", "memo0"):
            raise ValueError(f"ALTO_B200_MEMO_KERNEL must be fused or memo0, not {kind!r}")
        if kind == "fused" and (rank > 32 or nat.deterministic() or max(alto.shape.dims) >= 2**30):
            kind = "memo0"
        self.kind = kind
        self.fused = None
        g = _lanes(rank)
        fkey, ckey, ikey = ("fstream", m0, m1, g), ("memo_cons", m0, m1, g), ("memo_index", m0, m1)
        if kind == "fused" and fkey in alto._cache and ckey in alto._cache:
            # everything the fused pair runs on is cached: no piece index
            self.fused, self.cons = alto._cache[fkey], alto._cache[ckey]
            self.P = self.cons[4]
        else:
            # the view and piece index depend on the tensor only: built once
            # and cached on it (the fused pair drops them once its own
            # layouts exist: 20 B/nnz + 12 B/piece less); T belongs to the plan
            idx = alto._cache.get(ikey)
            if idx is None:
                if (kind == "fused" and fkey not in alto._cache and alto.nnz > 0
                        and nat.env_str("ALTO_B200_STREAM_BUILD", "fused").lower() != "legacy"):
                    # one pass: the stream (cached under fkey) and the view's
                    # (row, fiber) coordinates the piece index is built from;
                    # not cached as an index (no values, one coordinate plane)
                    idx = self._build_index(alto, m0, m1, fused_rank=rank)
                else:
                    idx = alto._cache[ikey] = self._build_index(alto, m0, m1)
            self.vals, self.rows, self.crd, self.pbase, self.prow, self.pcrd, self.pid, self.P = idx
        if kind == "fused" and self.fused is None:
            # the same stream serves the plain 3-mode MTTKRP of m0
            # (partition.device_fused_stream, cached under its key)
            fz = alto._cache.get(fkey)
            if fz is None:
                n = ctypes.c_int64(0)
                nat.call("alto_il_length", alto.nnz, rank, ctypes.byref(n))
                dev = nat.device()
                fz = (t.empty(n.value, dtype=t.int32, device=dev), t.empty(n.value, dtype=t.int32, device=dev),
                      t.empty(n.value, dtype=t.int32, device=dev), t.empty(n.value, dtype=t.float64, device=dev))
                nat.call("alto_memo_fused_stream", nat.ptr(self.rows), nat.ptr(self.crd[self.jplane]),
                         nat.ptr(self.crd[1 - self.jplane]), nat.ptr(self.vals), alto.nnz, rank, nat.ptr(fz[0]),
                         nat.ptr(fz[1]), nat.ptr(fz[2]), nat.ptr(fz[3]), nat.stream_ptr())
                alto._cache[fkey] = fz
            self.fused = fz
            # T rows at their consumer slots: the consumer streams them
            dev = nat.device()
            n = ctypes.c_int64(0)
            nat.call("alto_memo_consumer_length", self.P, rank, ctypes.byref(n))
            cprow = t.empty(n.value, dtype=t.int32, device=dev)
            cpcrd = t.empty(n.value, dtype=t.int32, device=dev)
            slot = t.empty(max(self.P, 1), dtype=t.int32, device=dev)
            nat.call("alto_memo_consumer_layout", nat.ptr(self.prow), nat.ptr(self.pcrd), nat.ptr(self.pid),
                     self.P, rank, nat.ptr(cprow), nat.ptr(cpcrd), nat.ptr(slot), nat.stream_ptr())
            pos = t.empty_like(fz[0])
            nat.call("alto_memo_fused_pos", nat.ptr(self.rows), nat.ptr(self.crd[self.jplane]), alto.nnz,
                     nat.ptr(self.pbase), nat.ptr(slot), rank, nat.ptr(pos), nat.stream_ptr())
            del slot
            self.cons = alto._cache[ckey] = (cprow, cpcrd, pos, n.value, self.P)
            alto._cache.pop(ikey, None)
            self.vals = self.rows = self.crd = self.pbase = self.prow = self.pcrd = self.pid = None
        if kind == "fused":
            # zeroed once: the producer writes only real pieces' slots and the
            # consumer streams the padding slots as exact zeros
            self.T = t.zeros((self.cons[3], nat.padded_ld(rank)), dtype=t.float64, device=nat.device())
        if self.T is None:
            self.T = t.empty((max(self.P, 1), nat.padded_ld(rank)), dtype=t.float64, device=nat.device())

    @staticmethod
    def _build_index(alto: AltoTensor, m0: int, m1: int, fused_rank: int | None = None):
        t = nat.torch()
        dev = nat.device()
        M = alto.nnz
        ix = types.SimpleNamespace()
        L = nat.layout_struct(alto.layout)
        # m0's stream sorted by (row, m1 coordinate), stable in ALTO order, decoded
        perm = t.empty(M, dtype=t.int64, device=dev)
        b = ctypes.c_size_t(0)
        nat.call("alto_mode_view_scratch_bytes", M, ctypes.byref(b))
        scratch = t.empty(b.value, dtype=t.uint8, device=dev)
        st = nat.stream_ptr()
        jplane = m1 if m1 < m0 else m1 - 1
        if fused_rank is not None:
            # alto_fused_stream_build: the interleaved producer stream and the
            # view's (row, fiber) coordinates in one pass after the sort
            n = ctypes.c_int64(0)
            nat.call("alto_il_length", M, fused_rank, ctypes.byref(n))
            fz = (t.empty(n.value, dtype=t.int32, device=dev), t.empty(n.value, dtype=t.int32, device=dev),
                  t.empty((1, n.value), dtype=t.int32, device=dev), t.empty(n.value, dtype=t.float64, device=dev))
            ix.rows = t.empty(M, dtype=t.int32, device=dev)
            jcrd = t.empty(M, dtype=t.int32, device=dev)
            nat.call("alto_fused_stream_build", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M, m0, m1,
                     fused_rank, nat.ptr(perm), nat.ptr(fz[0]), nat.ptr(fz[1]), nat.ptr(fz[2]), nat.ptr(fz[3]),
                     nat.ptr(ix.rows), nat.ptr(jcrd), nat.ptr(scratch), b.value, st)
            del scratch, perm
            alto._cache[("fstream", m0, m1, _lanes(fused_rank))] = fz
            ix.vals = None
            ix.crd = {jplane: jcrd}
        else:
            vkeys = t.empty_like(alto._keys)
            ix.vals = t.empty_like(alto._vals)
            nat.call("alto_fiber_view", ctypes.byref(L), nat.ptr(alto._keys), nat.ptr(alto._vals), M, m0, m1,
                     nat.ptr(perm), nat.ptr(vkeys), nat.ptr(ix.vals), nat.ptr(scratch), b.value, st)
            del scratch, perm
            ix.rows = t.empty(M, dtype=t.int32, device=dev)
            ix.crd = t.empty((2, (M + 7) & ~7), dtype=t.int32, device=dev)
            nat.call("alto_decode_view", ctypes.byref(L), nat.ptr(vkeys), M, m0, nat.ptr(ix.rows),
                     nat.ptr(ix.crd), st)
            del vkeys
            jcrd = ix.crd[jplane]
        nseg = (M + 511) // 512
        counts = t.empty(nseg, dtype=t.int32, device=dev)
        ix.pbase = t.empty(nseg + 1, dtype=t.int32, device=dev)
        nat.call("alto_memo_pieces_count", nat.ptr(ix.rows), nat.ptr(jcrd), M, nat.ptr(counts),
                 nat.ptr(ix.pbase), st)
        del counts
        P = int(ix.pbase[-1].item()) & 0xFFFFFFFF
        ix.P = P
        keys = t.empty(P, dtype=t.int64, device=dev)
        ids = t.empty(P, dtype=t.int64, device=dev)
        nat.call("alto_memo_sort_scratch_bytes", P, ctypes.byref(b))
        scratch = t.empty(b.value, dtype=t.uint8, device=dev)
        ix.prow = t.empty(P, dtype=t.int32, device=dev)
        ix.pcrd = t.empty(P, dtype=t.int32, device=dev)
        ix.pid = t.empty(P, dtype=t.int32, device=dev)
        nat.call("alto_memo_pieces_build", nat.ptr(ix.rows), nat.ptr(jcrd), M, nat.ptr(ix.pbase), P,
                 alto.shape.dims[m0], alto.shape.dims[m1], nat.ptr(keys), nat.ptr(ids), nat.ptr(scratch),
                 b.value, nat.ptr(ix.prow), nat.ptr(ix.pcrd), nat.ptr(ix.pid), st)
        del keys, ids, scratch
        return ix.vals, ix.rows, ix.crd, ix.pbase, ix.prow, ix.pcrd, ix.pid, P

    @staticmethod
    def bytes_needed(alto: AltoTensor, rank: int, pieces_estimate: int | None = None) -> int:
        """Device bytes of the plan (pieces bounded by nnz when unknown)."""
        M = alto.nnz
        P = M if pieces_estimate is None else pieces_estimate
        # views + the interleaved producer stream, index, T, build scratch
        return M * 40 + P * (12 + 8 * nat.padded_ld(rank)) + M * 32

    def mttkrp_m0(self, alto: AltoTensor, dfac, out) -> None:
        if self.fused is not None:
            out.zero_()
            aj, ak = dfac.mats[self.m1], dfac.mats[self.k]
            fr, fj, fk, fv = self.fused
            nat.call("alto_memo_fused", nat.ptr(fr), nat.ptr(fj), nat.ptr(fk), nat.ptr(fv), alto.nnz, nat.ptr(aj),
                     aj.stride(0), nat.ptr(ak), ak.stride(0), self.rank, None, nat.ptr(self.cons[2]),
                     nat.ptr(self.T), self.T.stride(0), nat.ptr(out), out.stride(0), nat.stream_ptr())
            self.t_valid = True
            return
        out.zero_()
        nat.call("alto_mttkrp_memo0", ctypes.byref(nat.layout_struct(alto.layout)), nat.ptr(self.rows),
                 nat.ptr(self.crd), nat.ptr(self.vals), alto.nnz, ctypes.byref(dfac.struct), self.m0, self.m1,
                 nat.ptr(self.pbase), nat.ptr(self.T), self.T.stride(0), nat.ptr(out),
                 out.stride(0), nat.stream_ptr())
        self.t_valid = True

    def mttkrp_m1(self, dfac, out) -> None:
        if not self.t_valid:
            raise RuntimeError("memoised partial sums are stale: run the m0 pass first")
        out.zero_()
        a = dfac.mats[self.m0]
        if self.fused is not None:
            cprow, cpcrd = self.cons[0], self.cons[1]
            nat.call("alto_memo_consume", nat.ptr(cprow), nat.ptr(cpcrd), nat.ptr(self.T), self.T.stride(0), self.P,
                     nat.ptr(a), a.stride(0), self.rank, nat.ptr(out), out.stride(0), nat.stream_ptr())
            return
        nat.call("alto_mttkrp_memo1", nat.ptr(self.prow), nat.ptr(self.pcrd), nat.ptr(self.pid), nat.ptr(self.T),
                 self.T.stride(0),
                 self.P, nat.ptr(a), a.stride(0), self.rank, nat.ptr(out), out.stride(0), nat.stream_ptr())


class CallMemo:
    """Dimension-tree reuse across public ``mttkrp()`` calls on a 3-mode
    tensor (the reference recomputes every call, pkg/src/alto/kernels.py:284-303).

    A user's own CP-ALS loop calls mttkrp for modes 0, 1, 2, 0, ... with the
    factor of the previous mode updated in between; the MTTKRPs of modes m
    and m + 1 then share T[i, j] = sum_k v A_k[k] (k = m + 2, unchanged
    between the two calls), exactly like the memoised sweep (MemoPlan). Once
    the calls follow the cyclic order (``MIN_STREAK`` consecutive steps), a
    call of mode m queues, on the device:

      1. ``alto_memo_key_check``: is A_{m+1} (just uploaded) bitwise equal to
         the A_k the previous mode's T was produced with?
      2. yes: the streaming consumer of that T (``alto_memo_consume_if``);
         no: the fused producer of mode m (``alto_memo_fused_if``), which
         stores T for mode m + 1, and ``alto_memo_key_save`` of its A_k.

    The choice never leaves the device (both kernels are queued, one returns
    at once); the flag comes back with the result, which the call reads
    anyway. T is a function of the tensor and A_k only, so a bitwise-equal
    key makes the consumer's result the same MTTKRP (to rounding, the order
    of the fp64 sums: the memoised sweep's 1e-12 bar). Numpy factors only
    (those calls synchronise before returning); ALTO_B200_CALL_MEMO=0 turns
    it off."""

    MIN_STREAK = 2

    def __init__(self, alto: AltoTensor, rank: int):
        t = nat.torch()
        self.alto, self.rank = alto, rank
        self.plans = {}
        self.keys = {}
        self.ready = set()
        self.flag = t.zeros(1, dtype=t.int32, device=nat.device())
        self.last = None
        self.streak = 0
        self.disabled = False
        self.stats = {"produce": 0, "consume": 0}

    @staticmethod
    def eligible(alto: AltoTensor, rank: int) -> bool:
        return (alto.ndim == 3 and rank <= 32 and not nat.deterministic() and max(alto.shape.dims) < 2**30
                and alto.nnz > 0 and nat.env_flag("ALTO_B200_CALL_MEMO", True)
                and nat.env_str("ALTO_B200_MEMO_KERNEL", "fused").lower() == "fused")

    def observe(self, mode: int) -> bool:
        """Record a call; True when the memo serves it."""
        if self.last is not None and mode == (self.last + 1) % 3:
            self.streak += 1
        else:
            self.streak = 0
        self.last = mode
        return not self.disabled and self.streak >= self.MIN_STREAK and self._fits(mode)

    def _fits(self, mode: int) -> bool:
        if mode in self.plans:
            return True
        t = nat.torch()
        try:
            free = t.cuda.mem_get_info()[0]
        except Exception:
            return False
        if MemoPlan.bytes_needed(self.alto, self.rank) > 0.5 * free:
            self.disabled = True
            return False
        return True

    def _plan(self, m0: int) -> MemoPlan:
        p = self.plans.get(m0)
        if p is None:
            p = MemoPlan(self.alto, self.rank, m0, (m0 + 1) % 3)
            if p.fused is None:
                raise RuntimeError("call memo needs the fused producer")
            self.plans[m0] = p
        return p

    def launch(self, dfac, mode: int, out) -> None:
        """Queue mode ``mode``'s MTTKRP into ``out`` (zeroed here)."""
        t = nat.torch()
        R = self.rank
        st = nat.stream_ptr()
        prev, k_prev = (mode - 1) % 3, (mode + 1) % 3
        prod = self._plan(mode)
        k = (mode + 2) % 3
        key = self.keys.get(mode)
        if key is None:
            key = self.keys[mode] = t.empty((self.alto.shape.dims[k], nat.padded_ld(R)), dtype=t.float64,
                                            device=nat.device())
        nat.call("alto_memset_async", nat.ptr(out), out.numel() * out.element_size(), st)
        cons_ok = prev in self.ready
        a_kp = dfac.mats[k_prev]
        kp = self.keys.get(prev)
        nat.call("alto_memo_key_check", nat.ptr(a_kp), a_kp.stride(0), nat.ptr(kp) if cons_ok else None,
                 kp.stride(0) if cons_ok else R, self.alto.shape.dims[k_prev], R, int(cons_ok), nat.ptr(self.flag),
                 st)
        if cons_ok:
            cons = self.plans[prev]
            a = dfac.mats[prev]
            cprow, cpcrd = cons.cons[0], cons.cons[1]
            nat.call("alto_memo_consume_if", nat.ptr(cprow), nat.ptr(cpcrd), nat.ptr(cons.T), cons.T.stride(0),
                     cons.P, nat.ptr(a), a.stride(0), R, nat.ptr(out), out.stride(0), nat.ptr(self.flag), 1, st)
        aj, ak = dfac.mats[(mode + 1) % 3], dfac.mats[k]
        fr, fj, fk, fv = prod.fused
        nat.call("alto_memo_fused_if", nat.ptr(fr), nat.ptr(fj), nat.ptr(fk), nat.ptr(fv), self.alto.nnz,
                 nat.ptr(aj), aj.stride(0), nat.ptr(ak), ak.stride(0), R, None, nat.ptr(prod.cons[2]),
                 nat.ptr(prod.T), prod.T.stride(0), nat.ptr(out), out.stride(0), nat.ptr(self.flag), 0, st)
        nat.call("alto_memo_key_save", nat.ptr(ak), ak.stride(0), nat.ptr(key), key.stride(0),
                 self.alto.shape.dims[k], R, nat.ptr(self.flag), 0, st)
        self._pending = mode

    def settle(self, consumed: bool) -> None:
        """After the call's sync: a producing call leaves a valid T + key."""
        mode = self._pending
        if consumed:
            self.stats["consume"] += 1
        else:
            self.stats["produce"] += 1
            self.ready.add(mode)


def call_memo(alto: AltoTensor, rank: int):
    """The tensor's CallMemo for ``rank`` (None when not eligible)."""
    if not CallMemo.eligible(alto, rank):
        return None
    key = ("callmemo", rank)
    cm = alto._cache.get(key)
    if cm is None:
        cm = alto._cache[key] = CallMemo(alto, rank)
    return cm
