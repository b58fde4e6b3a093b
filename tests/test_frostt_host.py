"""FROSTT text parse through the C ABI (host code, runs without a GPU):
error classes, messages and line numbers of pkg/src/alto/tensor.py:245-296
(the reference's own cases, pkg/tests/test_tensor.py:24-78), and a
multi-megabyte file parsed by several threads equal to numpy's parse."""

import ctypes

import numpy as np
import pytest

from paper_2403_06348_b200 import _native as nat


def _scan_parse(text: str, threads: int = 0):
    lib = nat.load()
    data = text.encode()
    e, n, err = ctypes.c_int64(0), ctypes.c_int32(0), ctypes.c_int64(-1)
    if lib.alto_frostt_scan(data, len(data), threads, ctypes.byref(e), ctypes.byref(n), ctypes.byref(err)):
        return None, None, (lib.alto_last_error().decode(), err.value)
    c = np.zeros((e.value, n.value), dtype=np.int64)
    v = np.zeros(e.value)
    if e.value and lib.alto_frostt_parse(data, len(data), threads, n.value, e.value,
                                         c.ctypes.data_as(ctypes.c_void_p),
                                         v.ctypes.data_as(ctypes.c_void_p), ctypes.byref(err)):
        return None, None, (lib.alto_last_error().decode(), err.value)
    return c, v, None


def test_basic_lines():
    c, v, e = _scan_parse("1 4 1 1.0\n")
    assert e is None and c.tolist() == [[0, 3, 0]] and v.tolist() == [1.0]
    c, v, e = _scan_parse("# hi\n\n  \n2 3 4.5\n")
    assert c.tolist() == [[1, 2]] and v.tolist() == [4.5]
    c, v, e = _scan_parse("1 1 1 2.5\n1 1 1 0.5\n")  # duplicates kept here, summed on the GPU
    assert c.tolist() == [[0, 0, 0]] * 2 and v.tolist() == [2.5, 0.5]
    c, v, e = _scan_parse("1\t2\t-3e-2\r\n+2 3 .5\r\n")
    assert c.tolist() == [[0, 1], [1, 2]] and v.tolist() == [-0.03, 0.5]


@pytest.mark.parametrize(
    "text,msg,line",
    [
        ("1 2\n1 2 3\n", "expected 2 fields, got 3", 2),
        ("a 2 3\n", "bad index in ['a', '2']", 1),
        ("0 2 3\n", "indices are one-based, got [0, 2]", 1),
        ("1 2 nan\n", "non-finite value 'nan'", 1),
        ("1 2 inf\n", "non-finite value 'inf'", 1),
        ("1 2 x\n", "bad value 'x'", 1),
        ("1 2 0x10\n", "bad value '0x10'", 1),
        ("1 1 1\n2 2 2\nbad line here\n", "bad index in ['bad', 'line']", 3),
        ("# c\n5\n", "expected at least one index and a value", 2),
    ],
)
def test_errors_match_reference(text, msg, line):
    _c, _v, e = _scan_parse(text)
    assert e == (msg, line)


def test_empty_inputs_have_no_entries():
    for text in ("", "# only comments\n", "\n\n"):
        c, v, e = _scan_parse(text)
        assert e is None and c.shape[0] == 0


def test_large_file_multithreaded_matches_numpy():
    rng = np.random.default_rng(0)
    M, N = 200_000, 4
    coords = rng.integers(1, 10**6, size=(M, N))
    vals = rng.standard_normal(M) * 10.0 ** rng.integers(-5, 5, size=M)
    lines = [" ".join(map(str, r)) + f" {v!r}\n" for r, v in zip(coords.tolist(), vals.tolist())]
    lines.insert(1000, "# a comment in the middle\n")
    lines.insert(70_000, "\n")
    text = "".join(lines)
    assert len(text) > 8 << 20  # several 1 MiB chunks
    for threads in (1, 3, 0):
        c, v, e = _scan_parse(text, threads)
        assert e is None
        assert np.array_equal(c, coords - 1)
        assert np.array_equal(v, vals)  # strtod and Python's float agree bit-for-bit
    bad = text.replace(lines[150_000], "1 2 3\n")
    _c, _v, e = _scan_parse(bad, 4)
    assert e == ("expected 5 fields, got 3", 150_001)  # lines[150_000] is file line 150001
