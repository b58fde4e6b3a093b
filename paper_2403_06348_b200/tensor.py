"""Device-resident sparse tensor containers and statistics.

``CooTensor`` (canonical coordinate list) and ``AltoTensor`` (sorted ALTO
positions + values) mirror pkg/src/alto/tensor.py:59-230, but their arrays
live in B200 HBM: canonicalisation (sort, duplicate merge, zero drop),
linearisation and sorting run as sm_100a kernels behind the C ABI. The numpy
views the reference exposes (``coords``, ``values``, ``positions``) are
materialised lazily on first access.

Statistics (``TensorStats``, ``compute_stats``, ``classify_reuse``) are host
arithmetic restated from pkg/src/alto/tensor.py:432-500.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native as nat
from .encoding import (
    UnsupportedShapeError,
    AltoLayout,
    TensorShape,
    alto_metadata_bits,
    as_shape,
    build_layout,
    coo_compression_ratio,
    lexicographic_layout,
    position_to_int,
    sfc_metadata_bits,
)

REUSE_LIMITED_BELOW = 5.0
REUSE_HIGH_ABOVE = 8.0


class ParseError(ValueError):
    """Malformed tensor text input (kept for API parity)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class AltoFormatError(ValueError):
    """Corrupt or unsupported binary tensor file (kept for API parity)."""


def _to_device(a, dtype):
    t = nat.torch()
    dev = nat.device()
    if isinstance(a, t.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return t.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def _keys_to_device(positions, word_bits: int):
    """Positions (numpy uint64 / torch int64 bit pattern) -> device int64."""
    t = nat.torch()
    if isinstance(positions, t.Tensor):
        keys = positions.to(device=nat.device())
        if keys.dtype != t.int64:
            keys = keys.view(t.int64) if keys.dtype == t.uint64 else keys.to(t.int64)
        return keys.contiguous()
    arr = np.ascontiguousarray(np.asarray(positions, dtype=np.uint64)).view(np.int64)
    return t.from_numpy(arr).to(nat.device())


def _sort_scratch(M: int, word_bits: int):
    b = ctypes.c_size_t(0)
    nat.call("alto_sort_scratch_bytes", max(M, 1), word_bits, ctypes.byref(b))
    t = nat.torch()
    return t.empty(b.value, dtype=t.uint8, device=nat.device())


def device_encode(layout: AltoLayout, dcoords):
    """(M, N) int64 device coords -> device keys (M,) or (M, 2) int64."""
    t = nat.torch()
    M = dcoords.shape[0]
    shape = (M,) if layout.word_bits == 64 else (M, 2)
    keys = t.empty(shape, dtype=t.int64, device=nat.device())
    bad = ctypes.c_int64(-1)
    rc = nat.load().alto_encode(
        ctypes.byref(nat.layout_struct(layout)), nat.ptr(dcoords), M, nat.ptr(keys),
        ctypes.byref(bad), nat.stream_ptr(),
    )
    if rc == nat.ALTO_ERR_INDEX:
        row = dcoords[bad.value].cpu().numpy()
        dims = np.asarray(layout.shape.dims)
        n = int(np.argmax((row < 0) | (row >= dims)))
        raise IndexError(f"coordinate {int(row[n])} out of range in mode {n}")
    nat.check(rc)
    return keys


def device_decode(layout: AltoLayout, keys):
    t = nat.torch()
    M = keys.shape[0]
    out = t.empty((M, layout.ndim), dtype=t.int64, device=nat.device())
    nat.call("alto_decode", ctypes.byref(nat.layout_struct(layout)), nat.ptr(keys), M,
             nat.ptr(out), nat.stream_ptr())
    return out


def encode_coords(layout: AltoLayout, coords) -> np.ndarray:
    """Array linearize (device kernel); numpy in, numpy out like
    pkg/src/alto/encoding.py:228-247."""
    coords = np.asarray(coords)
    if coords.ndim != 2 or coords.shape[1] != layout.ndim:
        raise ValueError(f"coords must be (M, {layout.ndim}), got {coords.shape}")
    keys = device_encode(layout, _to_device(coords.astype(np.int64), nat.torch().int64))
    out = keys.cpu().numpy().view(np.uint64)
    return out


def decode_coords(layout: AltoLayout, positions) -> np.ndarray:
    """Array delinearize (device kernel); pkg/src/alto/encoding.py:250-262."""
    keys = _keys_to_device(positions, layout.word_bits)
    if layout.word_bits == 128 and keys.ndim == 1:
        keys = keys.reshape(-1, 2)
    return device_decode(layout, keys).cpu().numpy()


# ---------------------------------------------------------------------------


class CooTensor:
    """Canonical coordinate-format sparse tensor (device resident).

    Construction validates ranges/finiteness, then sorts lexicographically,
    sums duplicates in input order and drops exact zeros on the GPU
    (pkg/src/alto/tensor.py:59-124)."""

    __slots__ = ("shape", "_dcoords", "_dvalues", "_coords", "_values")

    def __init__(self, shape, coords, values):
        t = nat.torch()
        shape = as_shape(shape)
        is_t = isinstance(coords, t.Tensor)
        cshape = tuple(coords.shape) if is_t else np.shape(np.asarray(coords, dtype=np.int64))
        if len(cshape) == 1 and cshape[0] == 0:
            cshape = (0, shape.ndim)
        if len(cshape) != 2 or cshape[1] != shape.ndim:
            raise ValueError(f"coords must have shape (M, {shape.ndim}), got {cshape}")
        vshape = tuple(values.shape) if isinstance(values, t.Tensor) else np.shape(
            np.asarray(values, dtype=np.float64))
        if vshape != (cshape[0],):
            raise ValueError("values must be a vector matching coords rows")
        M = cshape[0]
        dc = _to_device(coords if is_t else np.asarray(coords, dtype=np.int64).reshape(M, shape.ndim),
                        t.int64)
        dv = _to_device(values if isinstance(values, t.Tensor) else np.asarray(values, dtype=np.float64),
                        t.float64)
        if M:
            flags = (ctypes.c_int64 * 2)()
            dims = (ctypes.c_int64 * shape.ndim)(*shape.dims)
            nat.call("alto_validate_coo", nat.ptr(dc), nat.ptr(dv), M, shape.ndim, dims, flags,
                     nat.stream_ptr())
            if flags[0] >= 0:
                raise ValueError("coordinate out of range for shape")
            if flags[1] >= 0:
                raise ValueError("tensor values must be finite")
            dc, dv = _canonicalize(shape, dc, dv)
        self.shape = shape
        self._dcoords = dc
        self._dvalues = dv
        self._coords = None
        self._values = None

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None:
            self._coords = self._dcoords.cpu().numpy()
        return self._coords

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._dvalues.cpu().numpy()
        return self._values

    @property
    def nnz(self) -> int:
        return int(self._dvalues.shape[0])

    @property
    def ndim(self) -> int:
        return self.shape.ndim

    @classmethod
    def from_dense(cls, array) -> "CooTensor":
        array = np.asarray(array, dtype=np.float64)
        coords = np.argwhere(array != 0)
        return cls(array.shape, coords, array[tuple(coords.T)])

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape.dims, dtype=np.float64)
        out[tuple(self.coords.T)] = self.values
        return out

    def __eq__(self, other) -> bool:
        if not isinstance(other, CooTensor):
            return NotImplemented
        return (
            self.shape.dims == other.shape.dims
            and np.array_equal(self.coords, other.coords)
            and np.array_equal(self.values, other.values)
        )

    def __repr__(self) -> str:
        return f"CooTensor(shape={self.shape.dims}, nnz={self.nnz})"


def _canonicalize(shape: TensorShape, dcoords, dvalues):
    """Lexicographic sort + duplicate sum + zero drop, all on device: the
    coordinates are packed into lexicographic keys (mode 0 most significant),
    stably sorted carrying the input index, then each run of equal keys is
    summed sequentially in input order (np.add.at order)."""
    lex = lexicographic_layout(shape)
    keys = device_encode(lex, dcoords)
    vals = dvalues.clone()
    M = keys.shape[0]
    scratch = _sort_scratch(M, lex.word_bits)
    out_n = ctypes.c_int64(0)
    nat.call("alto_canonicalize", ctypes.byref(nat.layout_struct(lex)), nat.ptr(keys), nat.ptr(vals),
             M, nat.ptr(scratch), scratch.numel(), ctypes.byref(out_n), nat.stream_ptr())
    m = out_n.value
    keys = keys[:m].contiguous()
    return device_decode(lex, keys), vals[:m].contiguous()


class AltoTensor:
    """Nonzeros as sorted ALTO positions plus values, resident on the GPU.

    ``positions``/``values``/``coords`` are numpy views materialised on first
    access; kernels read the device arrays ``_keys`` (int64 bit patterns of
    the uint64 positions) and ``_vals``."""

    __slots__ = ("layout", "_keys", "_vals", "_positions", "_values", "_coords",
                 "_segments", "_views", "_cache")

    def __init__(self, layout: AltoLayout, positions, values, _validate: bool = True):
        t = nat.torch()
        if isinstance(positions, t.Tensor):
            pshape = tuple(positions.shape)
        else:
            pshape = np.shape(np.asarray(positions, dtype=np.uint64))
        vlen = (values.shape[0] if isinstance(values, t.Tensor)
                else np.asarray(values, dtype=np.float64).shape[0])
        if layout.word_bits == 64:
            if len(pshape) != 1:
                raise ValueError("64-bit layouts store positions as a flat array")
        elif len(pshape) != 2 or pshape[1] != 2:
            raise ValueError("128-bit layouts store positions as (M, 2) word pairs")
        if vlen != pshape[0]:
            raise ValueError("positions and values must have equal length")
        self.layout = layout
        self._keys = _keys_to_device(positions, layout.word_bits)
        self._vals = _to_device(values, t.float64)
        self._positions = None
        self._values = None
        self._coords = None
        self._segments = {}
        self._views = {}
        self._cache = {}
        if _validate:
            self._check_invariants()

    def _check_invariants(self):
        t = nat.torch()
        if self.nnz == 0:
            raise ValueError("linearized tensor must hold at least one nonzero")
        if not _strictly_increasing(self._keys):
            raise ValueError("positions must be strictly increasing")
        c = device_decode(self.layout, self._keys)
        dims = t.tensor(self.shape.dims, dtype=t.int64, device=c.device)
        if bool(((c < 0) | (c >= dims)).any()):
            raise ValueError("a position decodes outside the tensor shape")
        if not bool(t.isfinite(self._vals).all()):
            raise ValueError("tensor values must be finite")

    @property
    def shape(self) -> TensorShape:
        return self.layout.shape

    @property
    def ndim(self) -> int:
        return self.layout.ndim

    @property
    def nnz(self) -> int:
        return int(self._vals.shape[0])

    @property
    def positions(self) -> np.ndarray:
        if self._positions is None:
            self._positions = self._keys.cpu().numpy().view(np.uint64)
        return self._positions

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._vals.cpu().numpy()
        return self._values

    @property
    def coords(self) -> np.ndarray:
        """Decoded (M, N) coordinates (decoded on device, cached on host)."""
        if self._coords is None:
            self._coords = device_decode(self.layout, self._keys).cpu().numpy()
        return self._coords

    def device_coords(self):
        return device_decode(self.layout, self._keys)

    def position_ints(self) -> list[int]:
        p = self.positions
        if p.ndim == 1:
            return [int(v) for v in p]
        return [position_to_int(v) for v in p]

    @classmethod
    def from_coo(cls, coo: CooTensor, timings: dict | None = None) -> "AltoTensor":
        """Linearise on device, then radix-sort (key, value) pairs on device
        (pkg/src/alto/tensor.py:188-210)."""
        if coo.nnz == 0:
            raise ValueError("cannot linearize an empty tensor")
        t = nat.torch()
        t0 = time.perf_counter()
        layout = build_layout(coo.shape)
        keys = device_encode(layout, coo._dcoords)
        vals = coo._dvalues.clone()
        if timings is not None:
            t.cuda.synchronize()
        t1 = time.perf_counter()
        sort_pairs(layout, keys, vals)
        if timings is not None:
            t.cuda.synchronize()
        t2 = time.perf_counter()
        if timings is not None:
            timings["linearize_s"] = t1 - t0
            timings["sort_s"] = t2 - t1
        return cls(layout, keys, vals, _validate=False)

    @classmethod
    def from_device_coo(cls, shape, dcoords, dvalues, sort: bool = True) -> "AltoTensor":
        """Build from already-canonical device arrays (unique coordinates),
        skipping the CooTensor copy; used by the synthetic generators."""
        layout = build_layout(shape)
        keys = device_encode(layout, dcoords)
        vals = dvalues.to(nat.torch().float64).clone()
        if sort:
            sort_pairs(layout, keys, vals)
        return cls(layout, keys, vals, _validate=False)

    def to_coo(self) -> CooTensor:
        return CooTensor(self.shape, self.device_coords(), self._vals)

    def __repr__(self) -> str:
        return f"AltoTensor(shape={self.shape.dims}, nnz={self.nnz}, bits={self.layout.total_bits})"


# the onesweep radix sort packs look-back counts in 30 bits (csrc/radix_sort.cu)
MAX_SORT_NNZ = (1 << 30) - 1


def sort_pairs(layout: AltoLayout, keys, vals) -> None:
    M = vals.shape[0]
    if M > MAX_SORT_NNZ:
        raise UnsupportedShapeError(
            f"one GPU sorts at most 2^30 - 1 nonzeros ({M} given); build larger tensors with "
            "distributed.build_sharded, where every rank sorts only its own slice")
    scratch = _sort_scratch(M, layout.word_bits)
    nat.call("alto_sort_pairs", ctypes.byref(nat.layout_struct(layout)), nat.ptr(keys), nat.ptr(vals),
             M, nat.ptr(scratch), scratch.numel(), nat.stream_ptr())


def _strictly_increasing(keys) -> bool:
    t = nat.torch()
    if keys.shape[0] <= 1:
        return True
    flip = t.iinfo(t.int64).min  # xor the sign bit: signed order == unsigned order
    if keys.ndim == 1:
        k = keys ^ flip
        return bool((k[1:] > k[:-1]).all())
    hi, lo = keys[:, 1] ^ flip, keys[:, 0] ^ flip
    up = (hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))
    return bool(up.all())


def alto_from_coo(coo: CooTensor) -> AltoTensor:
    return AltoTensor.from_coo(coo)


def alto_to_coo(alto: AltoTensor) -> CooTensor:
    return alto.to_coo()


# ---------------------------------------------------------------------------
# statistics (pkg/src/alto/tensor.py:432-500)


@dataclass(frozen=True)
class TensorStats:
    shape: TensorShape
    nnz: int
    word_bits: int
    density: float
    fiber_reuse: tuple[float, ...]
    mode_classes: tuple[str, ...]
    overall_class: str
    s_coo_bits: int
    s_alto_bits: int
    s_sfc_bits: int
    compression_ratio: Fraction

    @classmethod
    def from_shape_nnz(cls, shape, nnz: int, word_bits: int = 64) -> "TensorStats":
        shape = as_shape(shape)
        if nnz < 1:
            raise ValueError("nnz must be positive")
        reuse = tuple(nnz / d for d in shape.dims)
        classes = tuple(classify_reuse(r) for r in reuse)
        coo_words = sum(-(-b // word_bits) for b in shape.mode_bits)
        return cls(
            shape=shape,
            nnz=nnz,
            word_bits=word_bits,
            density=nnz / math.prod(shape.dims),
            fiber_reuse=reuse,
            mode_classes=classes,
            overall_class=classes[int(np.argmin(reuse))],
            s_coo_bits=nnz * word_bits * coo_words,
            s_alto_bits=nnz * alto_metadata_bits(shape),
            s_sfc_bits=nnz * sfc_metadata_bits(shape),
            compression_ratio=coo_compression_ratio(shape, word_bits),
        )

    def to_json_dict(self) -> dict:
        return {
            "dims": list(self.shape.dims),
            "nnz": self.nnz,
            "word_bits": self.word_bits,
            "density": self.density,
            "fiber_reuse": list(self.fiber_reuse),
            "mode_classes": list(self.mode_classes),
            "overall_class": self.overall_class,
            "s_coo_bits": self.s_coo_bits,
            "s_alto_bits": self.s_alto_bits,
            "s_sfc_bits": self.s_sfc_bits,
            "compression_ratio": float(self.compression_ratio),
            "compression_ratio_exact": [
                self.compression_ratio.numerator,
                self.compression_ratio.denominator,
            ],
        }


def classify_reuse(reuse: float) -> str:
    if reuse < REUSE_LIMITED_BELOW:
        return "limited"
    if reuse <= REUSE_HIGH_ABOVE:
        return "medium"
    return "high"


def compute_stats(tensor, word_bits: int = 64) -> TensorStats:
    return TensorStats.from_shape_nnz(tensor.shape, tensor.nnz, word_bits)


# file formats live in io.py (device-direct loading); re-exported here so
# `from <pkg>.tensor import parse_frostt, read_alto, ...` works as in the
# reference (pkg/src/alto/tensor.py:245-412)
def parse_frostt(source, dims=None, **kw):
    from .io import parse_frostt as f

    return f(source, dims, **kw)


def write_frostt(coo, sink) -> None:
    from .io import write_frostt as f

    f(coo, sink)


def read_alto(source):
    from .io import read_alto as f

    return f(source)


def write_alto(alto, sink) -> None:
    from .io import write_alto as f

    f(alto, sink)
