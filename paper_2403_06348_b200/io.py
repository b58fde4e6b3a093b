"""Tensor files: the reference's binary ``.alto`` format and FROSTT text.

* ``write_alto`` / ``read_alto`` restate pkg/src/alto/tensor.py:326-412 (same
  byte layout, same header checks and error texts) with the payload moving
  straight between the file and HBM: ``read_alto`` reads positions and values
  in chunks into pinned host buffers and copies each chunk to the device
  while the next is read; the ALTO invariants are then checked on the GPU.
* ``parse_frostt`` restates pkg/src/alto/tensor.py:245-296: a multi-threaded
  host parse (``alto_frostt_scan`` / ``alto_frostt_parse`` in the C ABI) into
  pinned buffers, then the canonicalisation (lexicographic sort, duplicate
  sums in input order, zero drop) on the GPU through ``CooTensor``.
* ``write_frostt`` restates :299-308 (one-based indices, ``repr`` values).

Format::

    "ALTO" | u32 version | u8 word_bits | u8 ndim | u16 reserved
    | ndim * u64 dims | u64 nnz
    | total_bits * u8 schedule (mode id per line bit, LSB first)
    | nnz * position words (8 or 16 bytes each, little-endian)
    | nnz * f64 values (little-endian)
"""

from __future__ import annotations

import ctypes
import struct

from . import _native as nat
from .encoding import as_shape, layout_from_schedule
from .tensor import AltoFormatError, AltoTensor, CooTensor, ParseError

ALTO_MAGIC = b"ALTO"
ALTO_VERSION = 1
_CHUNK_BYTES = 64 << 20


def _open(target, mode: str):
    if hasattr(target, "read" if "r" in mode else "write"):
        return target, False
    return open(target, mode), True


def _pinned(nbytes: int):
    t = nat.torch()
    return t.empty(max(nbytes, 1), dtype=t.uint8, pin_memory=True)


# ---------------------------------------------------------------------------
# binary .alto


def write_alto(alto: AltoTensor, sink) -> None:
    """Header from the layout, then positions and values streamed from the
    device through a pinned chunk buffer."""
    t = nat.torch()
    stream, close = _open(sink, "wb")
    try:
        layout = alto.layout
        stream.write(ALTO_MAGIC)
        stream.write(struct.pack("<IBBH", ALTO_VERSION, layout.word_bits, layout.ndim, 0))
        stream.write(struct.pack(f"<{layout.ndim}Q", *layout.shape.dims))
        stream.write(struct.pack("<Q", alto.nnz))
        stream.write(bytes(mode for mode, _ in layout.schedule))
        for dev in (alto._keys, alto._vals):
            flat = dev.reshape(-1).view(t.uint8)
            buf = _pinned(min(flat.numel(), _CHUNK_BYTES))
            for off in range(0, flat.numel(), _CHUNK_BYTES):
                n = min(_CHUNK_BYTES, flat.numel() - off)
                buf[:n].copy_(flat[off:off + n])
                stream.write(memoryview(buf[:n].numpy()))
    finally:
        if close:
            stream.close()


def _unpack(data: bytes, offset: int, fmt: str):
    size = struct.calcsize(fmt)
    if len(data) - offset < size:
        raise AltoFormatError("truncated header")
    return struct.unpack_from(fmt, data, offset)


def _read_exact(stream, n: int) -> bytes:
    out = stream.read(n)
    return out if out is not None else b""


def read_alto(source) -> AltoTensor:
    """Parse and validate the header on the host, then load the payload
    directly into device memory (pinned double-buffered chunks)."""
    t = nat.torch()
    stream, close = _open(source, "rb")
    try:
        head = _read_exact(stream, 4 + 8)
        if head[:4] != ALTO_MAGIC:
            raise AltoFormatError("bad magic; not a linearized tensor file")
        version, word_bits, ndim, reserved = _unpack(head, 4, "<IBBH")
        if version != ALTO_VERSION:
            raise AltoFormatError(f"unsupported version {version}")
        if word_bits not in (64, 128):
            raise AltoFormatError(f"unsupported position width {word_bits}")
        if ndim < 1 or reserved != 0:
            raise AltoFormatError("corrupt header")
        more = _read_exact(stream, 8 * ndim + 8)
        dims = _unpack(more, 0, f"<{ndim}Q")
        (nnz,) = _unpack(more, 8 * ndim, "<Q")
        shape = as_shape(dims)
        total_bits = shape.total_bits
        if word_bits != (64 if total_bits <= 64 else 128):
            raise AltoFormatError("position width does not match the shape")
        mode_ids = _read_exact(stream, total_bits)
        if len(mode_ids) != total_bits:
            raise AltoFormatError("truncated schedule")
        ranks = [0] * ndim
        schedule = []
        for m in mode_ids:
            if m >= ndim:
                raise AltoFormatError(f"schedule names mode {m} of {ndim}")
            schedule.append((m, ranks[m]))
            ranks[m] += 1
        try:
            layout = layout_from_schedule(shape, schedule)
        except ValueError as exc:
            raise AltoFormatError(f"invalid schedule: {exc}") from None
        words = word_bits // 64
        payload = nnz * (8 * words + 8)
        # a corrupt or hostile header must not drive a device allocation:
        # bound nnz by the bytes the stream still holds when it can tell
        remaining = _remaining_bytes(stream)
        if remaining is not None and payload > remaining:
            raise AltoFormatError("truncated payload")
        dev = nat.device()
        try:
            keys = t.empty((nnz, 2) if words == 2 else (nnz,), dtype=t.int64, device=dev)
            vals = t.empty(nnz, dtype=t.float64, device=dev)
        except (RuntimeError, MemoryError) as exc:  # torch.cuda.OutOfMemoryError is a RuntimeError
            raise AltoFormatError(f"header announces {nnz} nonzeros: cannot allocate ({exc})") from None
        for target in (keys, vals):
            _load_into(stream, target.reshape(-1).view(t.uint8))
    finally:
        if close:
            stream.close()
    try:
        return AltoTensor(layout, keys, vals)
    except ValueError as exc:
        raise AltoFormatError(f"invariant violation: {exc}") from None


def _remaining_bytes(stream):
    """Bytes left in a seekable stream, else None."""
    try:
        if not stream.seekable():
            return None
        pos = stream.tell()
        end = stream.seek(0, 2)
        stream.seek(pos)
        return end - pos
    except (AttributeError, OSError, ValueError):
        return None


def _load_into(stream, dst) -> None:
    """Fill the device byte view ``dst`` from the stream: read a chunk into one
    pinned buffer while the previous one is being copied to the device."""
    t = nat.torch()
    total = dst.numel()
    if total == 0:
        return
    size = min(total, _CHUNK_BYTES)
    bufs = [_pinned(size), _pinned(size)]
    done = [None, None]
    off = 0
    i = 0
    while off < total:
        n = min(size, total - off)
        b = bufs[i]
        if done[i] is not None:
            done[i].synchronize()  # this buffer's previous copy has finished
        view = memoryview(b[:n].numpy())
        got = stream.readinto(view) if hasattr(stream, "readinto") else None
        if got is None:
            chunk = stream.read(n)
            got = len(chunk)
            view[:got] = chunk
        while got < n:  # short reads (pipes, BytesIO at the end)
            extra = stream.read(n - got)
            if not extra:
                break
            view[got:got + len(extra)] = extra
            got += len(extra)
        if got < n:
            raise AltoFormatError("truncated payload")
        dst[off:off + n].copy_(b[:n], non_blocking=True)
        ev = t.cuda.Event()
        ev.record()
        done[i] = ev
        off += n
        i ^= 1
    for ev in done:
        if ev is not None:
            ev.synchronize()


# ---------------------------------------------------------------------------
# FROSTT text


def _text_bytes(source) -> bytes:
    if hasattr(source, "read"):
        data = source.read()
        return data.encode() if isinstance(data, str) else bytes(data)
    with open(source, "rb") as f:
        return f.read()


def parse_frostt(source, dims=None, *, threads: int = 0) -> CooTensor:
    """FROSTT text -> canonical CooTensor: parallel host parse into pinned
    buffers, H2D, canonicalisation on the GPU."""
    t = nat.torch()
    data = _text_bytes(source)
    lib = nat.load()
    entries, ndim, err = ctypes.c_int64(0), ctypes.c_int32(0), ctypes.c_int64(-1)
    rc = lib.alto_frostt_scan(data, len(data), threads, ctypes.byref(entries), ctypes.byref(ndim),
                              ctypes.byref(err))
    if rc != nat.ALTO_OK:
        raise ParseError(lib.alto_last_error().decode(), err.value if err.value > 0 else None)
    M, N = entries.value, ndim.value
    if M == 0:
        raise ParseError("no nonzero entries found")
    coords = t.empty((M, N), dtype=t.int64, pin_memory=True)
    values = t.empty(M, dtype=t.float64, pin_memory=True)
    rc = lib.alto_frostt_parse(data, len(data), threads, N, M, ctypes.c_void_p(coords.data_ptr()),
                               ctypes.c_void_p(values.data_ptr()), ctypes.byref(err))
    if rc != nat.ALTO_OK:
        raise ParseError(lib.alto_last_error().decode(), err.value if err.value > 0 else None)
    dev = nat.device()
    dcoords = coords.to(dev, non_blocking=True)
    dvalues = values.to(dev, non_blocking=True)
    if dims is None:
        shape = as_shape((dcoords.max(dim=0).values + 1).cpu().tolist())
    else:
        shape = as_shape(dims)
        if shape.ndim != N:
            raise ParseError(f"file has {N} modes but dims has {shape.ndim}")
    coo = CooTensor(shape, dcoords, dvalues)
    if coo.nnz == 0:
        raise ParseError("tensor is empty after summing duplicates and dropping zeros")
    return coo


def write_frostt(coo: CooTensor, sink) -> None:
    """Canonical entries as one-based FROSTT text (round-trips parse)."""
    stream, close = _open(sink, "w")
    try:
        coords = coo.coords + 1
        lines = []
        for row, val in zip(coords.tolist(), coo.values.tolist()):
            lines.append(" ".join(map(str, row)) + f" {float(val)!r}\n")
        stream.write("".join(lines))
    finally:
        if close:
            stream.close()


__all__ = ["ALTO_MAGIC", "ALTO_VERSION", "parse_frostt", "read_alto", "write_alto", "write_frostt"]
