"""ctypes binding of libalto_b200.so (the C ABI in include/alto_b200.h).

This is the only door to the hot path: there is no CPU fallback. Loading
fails loudly when the library is missing, and every device entry requires a
CUDA device.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_size_t, c_uint8, c_void_p
from pathlib import Path

import numpy as np

from .encoding import (
    MAX_DEVICE_MODES,
    MAX_DEVICE_SPANS,
    AltoLayout,
    UnsupportedShapeError,
    word_spans,
)
from .validation import NumericalError

LIB_PATH = Path(os.environ.get("ALTO_B200_LIB") or Path(__file__).resolve().parent / "libalto_b200.so")

ALTO_OK = 0
ALTO_ERR_VALUE = 1
ALTO_ERR_INDEX = 2
ALTO_ERR_UNSUPPORTED = 3
ALTO_ERR_NUMERICAL = 4
ALTO_ERR_CUDA = 5

ALGO_ATOMIC = 0
ALGO_PRIVATIZED = 1


class LayoutStruct(ctypes.Structure):
    _fields_ = [
        ("nmodes", c_int32),
        ("word_bits", c_int32),
        ("total_bits", c_int32),
        ("nspans", c_int32),
        ("dims", c_int64 * MAX_DEVICE_MODES),
        ("span_off", c_int32 * (MAX_DEVICE_MODES + 1)),
        ("span_src", c_uint8 * MAX_DEVICE_SPANS),
        ("span_bit", c_uint8 * MAX_DEVICE_SPANS),
        ("span_len", c_uint8 * MAX_DEVICE_SPANS),
        ("span_word", c_uint8 * MAX_DEVICE_SPANS),
    ]


class FactorsStruct(ctypes.Structure):
    _fields_ = [
        ("nmodes", c_int32),
        ("rank", c_int32),
        ("ptr", c_void_p * MAX_DEVICE_MODES),
        ("ld", c_int64 * MAX_DEVICE_MODES),
    ]


# name -> argtypes (restype is always int)
_P = c_void_p
_SIGS = {
    "alto_abi_version": [],
    "alto_device_sm_count": [POINTER(c_int32)],
    "alto_encode": [POINTER(LayoutStruct), _P, c_int64, _P, POINTER(c_int64), _P],
    "alto_decode": [POINTER(LayoutStruct), _P, c_int64, _P, _P],
    "alto_sort_scratch_bytes": [c_int64, c_int32, POINTER(c_size_t)],
    "alto_sort_pairs": [POINTER(LayoutStruct), _P, _P, c_int64, _P, c_size_t, _P],
    "alto_canonicalize": [POINTER(LayoutStruct), _P, _P, c_int64, _P, c_size_t, POINTER(c_int64), _P],
    "alto_validate_coo": [_P, _P, c_int64, c_int32, POINTER(c_int64), POINTER(c_int64), _P],
    "alto_count_less": [c_int32, _P, c_int64, _P, c_int32, _P, _P],
    "alto_partition": [POINTER(LayoutStruct), _P, c_int64, c_int32, _P, _P, _P, _P],
    "alto_row_segment_span": [POINTER(LayoutStruct), _P, c_int64, c_int32, _P, c_int32, _P, _P, _P],
    "alto_mode_view": [POINTER(LayoutStruct), _P, _P, c_int64, c_int32, _P, _P, _P, _P, c_size_t, _P],
    "alto_mode_view_scratch_bytes": [c_int64, POINTER(c_size_t)],
    "alto_decode_view": [POINTER(LayoutStruct), _P, c_int64, c_int32, _P, _P, _P],
    "alto_mttkrp_dview": [POINTER(LayoutStruct), _P, _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                          c_int32, c_int32, _P, c_int64, _P],
    "alto_phi_dview": [POINTER(LayoutStruct), _P, _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                       c_int32, c_int32, _P, c_int64, _P, c_int64, c_double, _P, c_int64, _P, _P, _P],
    "alto_memo_pieces_count": [_P, _P, c_int64, _P, _P, _P],
    "alto_memo_sort_scratch_bytes": [c_int64, POINTER(c_size_t)],
    "alto_memo_pieces_build": [_P, _P, c_int64, _P, c_int64, c_int64, c_int64, _P, _P, _P, c_size_t, _P, _P, _P,
                               _P],
    "alto_mttkrp_memo0": [POINTER(LayoutStruct), _P, _P, _P, c_int64, POINTER(FactorsStruct), c_int32, c_int32,
                          _P, _P, c_int64, _P, c_int64, _P],
    "alto_gather_probe": [c_int32, c_int32, POINTER(c_double)],
    "alto_set_deterministic": [c_int32],
    "alto_get_deterministic": [POINTER(c_int32)],
    "alto_il_length": [c_int64, c_int32, POINTER(c_int64)],
    "alto_memo_fused_stream": [_P, _P, _P, _P, c_int64, c_int32, _P, _P, _P, _P, _P],
    "alto_memo_fused": [_P, _P, _P, _P, c_int64, _P, c_int64, _P, c_int64, c_int32, _P, _P, _P, c_int64, _P,
                        c_int64, _P],
    "alto_memo_consumer_length": [c_int64, c_int32, POINTER(c_int64)],
    "alto_memo_consumer_layout": [_P, _P, _P, c_int64, c_int32, _P, _P, _P, _P],
    "alto_memo_fused_pos": [_P, _P, c_int64, _P, _P, c_int32, _P, _P],
    "alto_memo_consume": [_P, _P, _P, c_int64, c_int64, _P, c_int64, c_int32, _P, c_int64, _P],
    "alto_memo_consume_if": [_P, _P, _P, c_int64, c_int64, _P, c_int64, c_int32, _P, c_int64, _P, c_int32, _P],
    "alto_memo_fused_if": [_P, _P, _P, _P, c_int64, _P, c_int64, _P, c_int64, c_int32, _P, _P, _P, c_int64, _P,
                           c_int64, _P, c_int32, _P],
    "alto_memo_key_check": [_P, c_int64, _P, c_int64, c_int64, c_int32, c_int32, _P, _P],
    "alto_memo_key_save": [_P, c_int64, _P, c_int64, c_int64, c_int32, _P, c_int32, _P],
    "alto_pstream_build_compact": [_P, _P, c_int64, _P, _P, _P],
    "alto_phi_pstream2": [_P, _P, c_int32, _P, c_int64, c_int32, c_int32, _P, c_int64, c_double, _P, c_int64, _P, _P],
    "alto_loglik_pstream2": [_P, _P, c_int32, _P, c_int64, c_int32, _P, c_int64, _P, c_int32, _P],
    "alto_fused_stream_n": [_P, _P, c_int64, c_int32, c_int32, _P, c_int64, c_int32, _P, _P, _P, _P, _P],
    "alto_fused_stream_build": [_P, _P, _P, c_int64, c_int32, c_int32, c_int32, _P, _P, _P, _P, _P, _P, _P, _P, c_size_t,
                                _P],
    "alto_mttkrp_fused": [_P, _P, _P, _P, c_int64, c_int32, _P, c_int64, _P, _P, c_int32, _P, c_int64, _P],
    "alto_mttkrp_memo1": [_P, _P, _P, _P, c_int64, c_int64, _P, c_int64, c_int32, _P, c_int64, _P],
    "alto_pstream_sizes": [c_int64, c_int32, POINTER(c_int64), POINTER(c_int64)],
    "alto_pstream_build": [_P, _P, c_int64, _P, _P, _P],
    "alto_loglik_pstream_partials": [POINTER(c_int32)],
    "alto_loglik_pstream": [_P, _P, _P, c_int64, c_int32, _P, c_int64, _P, c_int32, _P],
    "alto_phi_pstream": [_P, _P, _P, c_int64, c_int32, c_int32, _P, c_int64, c_double, _P, c_int64, _P, _P],
    "alto_pi_dview": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32, _P, c_int64, _P],
    "alto_loglik_dview_partials": [c_int64, c_int32, POINTER(c_int32)],
    "alto_loglik_dview": [POINTER(LayoutStruct), _P, _P, _P, c_int64, POINTER(FactorsStruct), c_int32, _P,
                          c_int64, _P, _P],
    "alto_blocked_view": [POINTER(LayoutStruct), _P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, _P,
                          _P, _P, c_size_t, _P],
    "alto_apr_inner_state_bytes": [c_int32, POINTER(c_size_t)],
    "alto_apr_inner_reset": [_P, _P],
    "alto_apr_inner_kkt_offset": [POINTER(c_size_t)],
    "alto_zero_if": [_P, c_int64, c_int64, _P, _P],
    "alto_copy_if": [_P, _P, c_int64, _P, _P],
    "alto_apr_inner_step": [_P, c_int64, _P, c_int64, c_int64, c_int32, c_double, c_int32, _P, _P],
    "alto_apr_inner_result": [_P, POINTER(c_int32), POINTER(c_int32), POINTER(c_double), _P],
    "alto_fiber_view": [POINTER(LayoutStruct), _P, _P, c_int64, c_int32, c_int32, _P, _P, _P, _P,
                        c_size_t, _P],
    "alto_mttkrp_stream": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                           _P, c_int64, c_int32, _P, _P, c_int32, _P],
    "alto_segment_smem_bytes": [c_int32, c_int32, c_int32, c_int64, POINTER(c_size_t)],
    "alto_mttkrp_segment": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                            _P, c_int64, _P, _P, c_int32, c_int64, c_int32, _P],
    "alto_mttkrp_exact": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                          _P, c_int64, _P, _P, _P, _P, c_int32, _P, _P],
    "alto_mttkrp_oriented": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                             _P, c_int64, c_int64, c_int32, _P, c_size_t, _P],
    "alto_run_scratch_bytes": [c_int64, POINTER(c_size_t)],
    "alto_default_segments": [c_int64, POINTER(c_int64)],
    "alto_pi": [POINTER(LayoutStruct), _P, c_int64, POINTER(FactorsStruct), c_int32, _P, c_int64, _P],
    "alto_phi_stream": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                        _P, c_int64, _P, c_int64, c_double, _P, c_int64, c_int32, _P, _P, c_int32, _P],
    "alto_phi_exact": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                       _P, c_int64, _P, c_int64, c_double, _P, c_int64, _P, _P, _P, _P, c_int32,
                       _P, _P],
    "alto_phi_oriented": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32,
                          _P, c_int64, _P, c_int64, c_double, _P, c_int64, c_int64, c_int32, _P,
                          c_size_t, _P],
    "alto_apr_update": [_P, c_int64, _P, c_int64, c_int64, c_int32, c_double, c_int32,
                        POINTER(c_double), _P],
    "alto_loglik": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), _P, _P,
                    POINTER(c_double), _P],
    "alto_loglik_partials": [c_int64, POINTER(c_int32)],
    "alto_als_update_scratch_bytes": [c_int64, c_int32, POINTER(c_size_t)],
    "alto_als_update": [_P, c_int64, c_int64, c_int32, _P, c_int32, c_int32, _P, c_int64, _P, _P, c_size_t,
                        _P, _P],
    "alto_als_solve_gram": [_P, c_int64, c_int64, c_int32, _P, c_int32, c_int32, _P, c_int64, _P, c_size_t, _P,
                            c_int32, _P, _P],
    "alto_als_normalize": [_P, c_int32, _P, c_int32, c_int32, _P, c_int64, c_int64, _P, _P, c_size_t, _P],
    "alto_als_chol": [_P, c_int32, c_int32, c_int32, _P, c_size_t, _P, _P],
    "alto_als_update_solve": [_P, c_int64, c_int64, c_int32, _P, c_int32, c_int32, _P, c_int64, _P, _P, c_size_t,
                              _P, c_int32, _P],
    "alto_factors_nonfinite": [POINTER(FactorsStruct), POINTER(c_int64), c_int32, _P, _P],
    "alto_upload_factors": [POINTER(FactorsStruct), _P, POINTER(c_int64), c_int32, c_int32, _P, _P],
    "alto_memset_async": [_P, c_size_t, _P],
    "alto_frostt_scan": [c_char_p, c_int64, c_int32, POINTER(c_int64), POINTER(c_int32), POINTER(c_int64)],
    "alto_frostt_parse": [c_char_p, c_int64, c_int32, c_int32, c_int64, _P, _P, POINTER(c_int64)],
    "alto_nccl_version": [POINTER(c_int32)],
    "alto_nccl_unique_id": [_P, c_int64],
    "alto_nccl_comm_init": [_P, c_int64, c_int32, c_int32, POINTER(c_void_p)],
    "alto_nccl_comm_destroy": [_P, c_int32],
    "alto_nccl_comm_info": [_P, POINTER(c_int32), POINTER(c_int32)],
    "alto_nccl_check": [_P],
    "alto_nccl_allreduce_f64": [_P, c_int64, _P, _P],
    "alto_nccl_reduce_scatter_f64": [_P, _P, c_int64, _P, _P],
    "alto_nccl_allgather_f64": [_P, _P, c_int64, _P, _P],
    "alto_mttkrp_sharded": [POINTER(LayoutStruct), _P, _P, c_int64, POINTER(FactorsStruct), c_int32, _P, c_int64,
                            c_int64, _P, _P, c_int32, c_int64, c_int32, c_int32, _P, _P],
}

EXPORTED = tuple(_SIGS) + ("alto_last_error",)

_lib = None


def load():
    """Load the library (raising if it is absent) and bind signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2403_06348_b200.build` "
            "(the ALTO hot path has no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int32
    lib.alto_last_error.argtypes = []
    lib.alto_last_error.restype = ctypes.c_char_p
    _lib = lib
    if env_flag("ALTO_B200_DETERMINISTIC"):
        lib.alto_set_deterministic(1)
    return lib


def set_deterministic(on: bool) -> None:
    """Bitwise run-to-run reproducible fast kernels (csrc/det.cu): edge runs
    of the decoded-view and memoised kernels are folded in a fixed order;
    decoded views are built unblocked. ``ALTO_B200_DETERMINISTIC=1`` sets it
    at load."""
    call("alto_set_deterministic", 1 if on else 0)


def deterministic() -> bool:
    v = ctypes.c_int32(0)
    call("alto_get_deterministic", ctypes.byref(v))
    return bool(v.value)


def check(rc: int) -> None:
    if rc == ALTO_OK:
        return
    msg = load().alto_last_error().decode(errors="replace")
    if rc == ALTO_ERR_VALUE:
        raise ValueError(msg)
    if rc == ALTO_ERR_INDEX:
        raise IndexError(msg)
    if rc == ALTO_ERR_UNSUPPORTED:
        raise UnsupportedShapeError(msg)
    if rc == ALTO_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


# ---------------------------------------------------------------------------
# device plumbing (torch provides memory and streams only)


def torch():
    import torch as _t

    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "the ALTO B200 hot path requires a CUDA device; there is no CPU fallback"
        )
    return t.device("cuda", t.cuda.current_device())


def stream_ptr():
    return c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t) -> c_void_p:
    return c_void_p(t.data_ptr()) if t is not None else c_void_p(0)


_LAYOUT_CACHE: dict = {}


def layout_struct(layout: AltoLayout) -> LayoutStruct:
    """Packed alto_layout_t for a layout (memoised per layout object; the
    struct is read-only for the C side)."""
    hit = _LAYOUT_CACHE.get(id(layout))
    if hit is not None and hit[0] is layout:
        return hit[1]
    s = _pack_layout(layout)
    if len(_LAYOUT_CACHE) > 256:
        _LAYOUT_CACHE.clear()
    _LAYOUT_CACHE[id(layout)] = (layout, s)
    return s


def _pack_layout(layout: AltoLayout) -> LayoutStruct:
    if layout.ndim > MAX_DEVICE_MODES:
        raise UnsupportedShapeError(
            f"device kernels support up to {MAX_DEVICE_MODES} modes, got {layout.ndim}"
        )
    s = LayoutStruct()
    s.nmodes = layout.ndim
    s.word_bits = layout.word_bits
    s.total_bits = layout.total_bits
    parts = word_spans(layout)
    k = 0
    for n in range(layout.ndim):
        s.dims[n] = layout.shape.dims[n]
        s.span_off[n] = k
        for src, bit, ln, word in parts[n]:
            if k >= MAX_DEVICE_SPANS:
                raise UnsupportedShapeError("layout has too many bit spans for the device table")
            s.span_src[k], s.span_bit[k], s.span_len[k], s.span_word[k] = src, bit, ln, word
            k += 1
    for n in range(layout.ndim, MAX_DEVICE_MODES + 1):
        s.span_off[n] = k
    s.nspans = k
    return s


def padded_ld(rank: int) -> int:
    """Row stride used on device (doubles): rows never straddle a 128-byte
    line more than their size requires -- 4 or 8 for short rows (32/64 B,
    sector aligned), else a multiple of 16 (128-B aligned rows). A gathered
    R = 10 row (80 B) then touches one L1 line instead of 1.5 on average
    (96-B stride), which is what the gather-bound kernels pay for."""
    if rank <= 4:
        return 4
    if rank <= 8:
        return 8
    return (rank + 15) // 16 * 16


def to_device_matrix(a, ld: int | None = None, non_blocking: bool = False):
    """Copy/convert a (rows, rank) matrix to a device float64 tensor whose row
    stride is ld (zero padding). Device tensors that already match are used
    as-is (no copy). ``non_blocking``: stream-ordered upload (a DMA straight
    from pinned host memory; pageable sources are staged by the driver before
    the call returns, so the host buffer may be reused either way)."""
    t = torch()
    dev = device()
    rows, rank = a.shape
    ld = padded_ld(rank) if ld is None else ld
    if isinstance(a, t.Tensor) and a.is_cuda and a.dtype == t.float64:
        if a.stride() == (ld, 1) and a.data_ptr() % 32 == 0:
            return a
    src = a if isinstance(a, t.Tensor) else t.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    out = (t.empty if ld == rank else t.zeros)((rows, ld), dtype=t.float64, device=dev)
    out[:, :rank].copy_(src, non_blocking=non_blocking)
    return out


def factors_struct(mats, rank: int) -> FactorsStruct:
    """mats: device float64 tensors (rows, ld) with ld >= rank."""
    s = FactorsStruct()
    s.nmodes = len(mats)
    s.rank = rank
    for n, m in enumerate(mats):
        s.ptr[n] = m.data_ptr()
        s.ld[n] = m.stride(0)
    return s


def sm_count() -> int:
    v = c_int32(0)
    call("alto_device_sm_count", ctypes.byref(v))
    return v.value


def default_segments(M: int) -> int:
    v = c_int64(0)
    call("alto_default_segments", M, ctypes.byref(v))
    return v.value


def run_scratch(nseg: int):
    b = c_size_t(0)
    call("alto_run_scratch_bytes", nseg, ctypes.byref(b))
    return torch().empty(b.value, dtype=torch().uint8, device=device())


_capture_stream = None


class graph_capture:
    """``torch.cuda.graph`` without its ``empty_cache()`` and pinned-host
    cache flush: those cost 6-8 ms per capture (a fifth of a warm 10-iteration
    ``cp_als`` on c2, tools/cold_als_prof.py) and drop the pinned buffers the
    public numpy path reuses. Same capture stream handling and error mode."""

    def __init__(self, cuda_graph):
        self.cuda_graph = cuda_graph

    def __enter__(self):
        global _capture_stream
        t = torch()
        if _capture_stream is None:
            _capture_stream = t.cuda.Stream()
        t.cuda.synchronize()
        if env_flag("ALTO_B200_GRAPH_EMPTY_CACHE", False):
            t.cuda.empty_cache()
        self._ctx = t.cuda.stream(_capture_stream)
        self._ctx.__enter__()
        self.cuda_graph.capture_begin()

    def __exit__(self, *args):
        self.cuda_graph.capture_end()
        self._ctx.__exit__(*args)


def env_str(name: str, default: str = "") -> str:
    v = os.environ.get(name)
    return default if v is None or not v.strip() else v.strip()


def env_flag(name: str, default: bool = False) -> bool:
    v = os.environ.get(name)
    if v is None:
        return default
    return v.strip().lower() not in ("", "0", "false", "no", "off")
