"""ALTO bit layout (host side) and the device-facing span tables.

The layout is O(total_bits) host logic; everything per-nonzero (encode,
decode, sort) runs on the GPU through the C-ABI in ``_native``.

Reference behaviour restated here (not copied):

* ``_mode_bits``            -- pkg/src/alto/encoding.py:32-34
* ``TensorShape``           -- pkg/src/alto/encoding.py:37-72 (128-bit cap :49-53)
* ``AltoLayout``            -- pkg/src/alto/encoding.py:90-114 (word_bits :108-110)
* ``build_layout``          -- pkg/src/alto/encoding.py:161-176
* ``layout_from_schedule``  -- pkg/src/alto/encoding.py:131-158
* span runs                 -- pkg/src/alto/encoding.py:117-128
* word-edge split           -- pkg/src/alto/encoding.py:213-225
* scalar linearize/delinearize -- pkg/src/alto/encoding.py:179-205
* storage formulas          -- pkg/src/alto/encoding.py:277-307
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Iterable, Sequence

import numpy as np

MAX_LINE_BITS = 128

_SUPPORTED_WORD_BITS = (8, 16, 32, 64)

# device-side limits (see include/alto_b200.h)
MAX_DEVICE_MODES = 16
MAX_DEVICE_SPANS = 192


class UnsupportedShapeError(ValueError):
    """Tensor shape cannot be linearized within the 128-bit position limit."""


def _mode_bits(dim: int) -> int:
    return 0 if dim <= 1 else int(dim - 1).bit_length()


@dataclass(frozen=True)
class TensorShape:
    """Mode lengths of a tensor plus derived per-mode bit widths."""

    dims: tuple[int, ...]

    def __init__(self, dims: Iterable[int]):
        dims = tuple(int(d) for d in dims)
        if not dims:
            raise ValueError("tensor must have at least one mode")
        if min(dims) < 1:
            raise ValueError(f"mode lengths must be >= 1, got {dims}")
        need = sum(_mode_bits(d) for d in dims)
        if need > MAX_LINE_BITS:
            raise UnsupportedShapeError(
                f"shape {dims} needs {need} index bits; the limit is {MAX_LINE_BITS}"
            )
        object.__setattr__(self, "dims", dims)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def mode_bits(self) -> tuple[int, ...]:
        return tuple(_mode_bits(d) for d in self.dims)

    @property
    def total_bits(self) -> int:
        return sum(self.mode_bits)

    def __iter__(self):
        return iter(self.dims)

    def __len__(self):
        return len(self.dims)


def as_shape(shape) -> TensorShape:
    return shape if isinstance(shape, TensorShape) else TensorShape(shape)


@dataclass(frozen=True)
class BitSpan:
    """``length`` consecutive bits: mode-index bit ``src`` <-> line bit ``dst``."""

    src: int
    dst: int
    length: int


@dataclass(frozen=True)
class AltoLayout:
    """LSB-first schedule of (mode, bit_rank), per-mode masks and spans."""

    shape: TensorShape
    schedule: tuple[tuple[int, int], ...]
    masks: tuple[int, ...] = field(repr=False)
    spans: tuple[tuple[BitSpan, ...], ...] = field(repr=False)

    @property
    def total_bits(self) -> int:
        return len(self.schedule)

    @property
    def word_bits(self) -> int:
        return 64 if self.total_bits <= 64 else 128

    @property
    def ndim(self) -> int:
        return self.shape.ndim


def _runs(schedule: Sequence[tuple[int, int]], ndim: int):
    """Group the schedule into maximal runs where both the line bit and the
    mode bit advance by one (so a run is one shift+mask)."""
    per_mode: list[list[list[int]]] = [[] for _ in range(ndim)]
    for dst, (mode, rank) in enumerate(schedule):
        runs = per_mode[mode]
        if runs:
            src0, dst0, ln = runs[-1]
            if src0 + ln == rank and dst0 + ln == dst:
                runs[-1][2] = ln + 1
                continue
        runs.append([rank, dst, 1])
    return tuple(tuple(BitSpan(*r) for r in runs) for runs in per_mode)


def layout_from_schedule(shape, schedule: Sequence[tuple[int, int]]) -> AltoLayout:
    """Validate an explicit LSB-first schedule and derive masks/spans."""
    shape = as_shape(shape)
    schedule = tuple((int(m), int(r)) for m, r in schedule)
    ranks: list[list[int]] = [[] for _ in range(shape.ndim)]
    for mode, rank in schedule:
        if mode < 0 or mode >= shape.ndim:
            raise ValueError(f"schedule names mode {mode} outside 0..{shape.ndim - 1}")
        ranks[mode].append(rank)
    bits = shape.mode_bits
    for n in range(shape.ndim):
        if ranks[n] != list(range(bits[n])):
            raise ValueError(
                f"mode {n} must contribute bit ranks 0..{bits[n] - 1} "
                f"in increasing order, got {ranks[n]}"
            )
    masks = [0] * shape.ndim
    for dst, (mode, _rank) in enumerate(schedule):
        masks[mode] |= 1 << dst
    return AltoLayout(shape, schedule, tuple(masks), _runs(schedule, shape.ndim))


def build_layout(shape) -> AltoLayout:
    """Adaptive interleave: group g holds bit g of every mode with > g bits,
    shortest mode at the low end of the group (ties: lower mode index)."""
    shape = as_shape(shape)
    bits = shape.mode_bits
    by_length = sorted(range(shape.ndim), key=lambda n: (shape.dims[n], n))
    schedule = [
        (n, g) for g in range(max(bits, default=0)) for n in by_length if bits[n] > g
    ]
    return layout_from_schedule(shape, schedule)


def lexicographic_layout(shape) -> AltoLayout:
    """Concatenated layout, mode 0 most significant: numeric order of these
    keys is the lexicographic coordinate order used by CooTensor
    canonicalisation (pkg/src/alto/tensor.py:116-124, np.unique(axis=0))."""
    shape = as_shape(shape)
    schedule = []
    for n in reversed(range(shape.ndim)):
        schedule.extend((n, r) for r in range(shape.mode_bits[n]))
    return layout_from_schedule(shape, schedule)


def linearize(layout: AltoLayout, coords: Sequence[int]) -> int:
    """Scalar bit gather (Python int)."""
    dims = layout.shape.dims
    if len(coords) != len(dims):
        raise ValueError(f"expected {len(dims)} coordinates, got {len(coords)}")
    pos = 0
    for n, (i, d) in enumerate(zip(coords, dims)):
        i = int(i)
        if i < 0 or i >= d:
            raise IndexError(f"coordinate {i} out of range [0, {d}) in mode {n}")
        for s in layout.spans[n]:
            pos |= ((i >> s.src) & ((1 << s.length) - 1)) << s.dst
    return pos


def delinearize(layout: AltoLayout, pos: int) -> tuple[int, ...]:
    """Scalar bit scatter (Python int)."""
    pos = int(pos)
    if pos < 0 or pos >= (1 << layout.total_bits):
        raise ValueError(f"position {pos} exceeds the {layout.total_bits}-bit line")
    return tuple(
        sum(((pos >> s.dst) & ((1 << s.length) - 1)) << s.src for s in layout.spans[n])
        for n in range(layout.ndim)
    )


def position_to_int(position) -> int:
    arr = np.asarray(position, dtype=np.uint64)
    if arr.ndim == 0:
        return int(arr)
    return int(arr[0]) | (int(arr[1]) << 64)


def word_spans(layout: AltoLayout) -> list[list[tuple[int, int, int, int]]]:
    """Per mode: (src, bit_in_word, length, word) with no span crossing a
    64-bit word edge -- the table the device encode/decode walks."""
    out = []
    for n in range(layout.ndim):
        parts = []
        for s in layout.spans[n]:
            src, dst, ln = s.src, s.dst, s.length
            while ln:
                word, bit = divmod(dst, 64)
                take = min(ln, 64 - bit)
                parts.append((src, bit, take, word))
                src, dst, ln = src + take, dst + take, ln - take
        out.append(parts)
    return out


# ---------------------------------------------------------------------------
# storage formulas (reporting only; pkg/src/alto/encoding.py:277-307)


def alto_metadata_bits(shape) -> int:
    return as_shape(shape).total_bits


def sfc_metadata_bits(shape) -> int:
    shape = as_shape(shape)
    return shape.ndim * max(shape.mode_bits)


def coo_compression_ratio(shape, word_bits: int = 64) -> Fraction:
    shape = as_shape(shape)
    if word_bits not in _SUPPORTED_WORD_BITS:
        raise ValueError(f"word_bits must be one of {_SUPPORTED_WORD_BITS}")
    coo_words = sum(-(-b // word_bits) for b in shape.mode_bits)
    alto_words = -(-shape.total_bits // word_bits)
    return Fraction(1) if alto_words == 0 else Fraction(coo_words, alto_words)
