"""FROSTT text and binary .alto files through the GPU path, mirroring the
reference's own cases (pkg/tests/test_tensor.py:24-205): parse semantics,
canonical merge on the device, header layout byte for byte, every header
error, invariant checks after the direct-to-device load, 128-bit files, and
text round trips."""

import io

import numpy as np
import pytest

import paper_2403_06348_b200 as alto
from conftest import EXAMPLE_COORDS, EXAMPLE_DIMS, EXAMPLE_VALUES, random_sparse
from paper_2403_06348_b200.tensor import parse_frostt as tensor_parse_frostt

pytestmark = pytest.mark.gpu

EXAMPLE_TNS = "# 4x8x2 example tensor\n" + "".join(
    " ".join(str(i + 1) for i in c) + f" {int(v)}\n" for c, v in zip(EXAMPLE_COORDS, EXAMPLE_VALUES))


@pytest.fixture(scope="module")
def example_coo():
    return alto.parse_frostt(io.StringIO(EXAMPLE_TNS), dims=EXAMPLE_DIMS)


@pytest.fixture(scope="module")
def example_alto(example_coo):
    return alto.AltoTensor.from_coo(example_coo)


class TestParse:
    def test_single_line(self):
        coo = alto.parse_frostt(io.StringIO("1 4 1 1.0\n"))
        assert coo.coords.tolist() == [[0, 3, 0]] and coo.values.tolist() == [1.0]

    def test_duplicates_summed(self):
        coo = alto.parse_frostt(io.StringIO("1 1 1 2.5\n1 1 1 0.5\n"))
        assert coo.nnz == 1 and coo.values.tolist() == [3.0]

    def test_zero_after_merge_dropped(self):
        with pytest.raises(alto.ParseError, match="empty"):
            alto.parse_frostt(io.StringIO("1 1 2\n1 1 -2\n"))

    def test_example_with_dims(self, example_coo):
        assert example_coo.nnz == 6 and example_coo.shape.dims == (4, 8, 2)

    def test_shape_inference_is_max_index(self):
        assert alto.parse_frostt(io.StringIO(EXAMPLE_TNS)).shape.dims == (4, 7, 2)

    def test_comments_and_blanks(self):
        assert alto.parse_frostt(io.StringIO("# hi\n\n  \n2 3 4.5\n")).shape.dims == (2, 3)

    @pytest.mark.parametrize("text,match", [
        ("1 2\n1 2 3\n", "fields"), ("a 2 3\n", "index"), ("0 2 3\n", "one-based"),
        ("1 2 nan\n", "non-finite"), ("1 2 inf\n", "non-finite"), ("1 2 x\n", "value"),
        ("", "no nonzero"), ("# only comments\n", "no nonzero")])
    def test_malformed(self, text, match):
        with pytest.raises(alto.ParseError, match=match):
            alto.parse_frostt(io.StringIO(text))

    def test_dims_must_match_modes(self):
        with pytest.raises(alto.ParseError, match="modes"):
            alto.parse_frostt(io.StringIO("1 2 3 4\n"), dims=(4, 4))

    def test_dims_too_small(self):
        with pytest.raises(ValueError):
            alto.parse_frostt(io.StringIO("9 1 1.0\n"), dims=(4, 4))

    def test_line_numbers_reported(self):
        with pytest.raises(alto.ParseError, match="line 3"):
            alto.parse_frostt(io.StringIO("1 1 1\n2 2 2\nbad line here\n"))

    def test_tensor_module_reexport_and_paths(self, tmp_path):
        p = tmp_path / "t.tns"
        p.write_text(EXAMPLE_TNS)
        assert tensor_parse_frostt(str(p), dims=EXAMPLE_DIMS) == alto.parse_frostt(p, dims=EXAMPLE_DIMS)


class TestBinaryFormat:
    def test_roundtrip(self, example_alto, example_coo, tmp_path):
        path = tmp_path / "t.alto"
        alto.write_alto(example_alto, str(path))
        back = alto.read_alto(str(path))
        assert back.to_coo() == example_coo
        assert back.layout.schedule == example_alto.layout.schedule
        assert back.position_ints() == [2, 15, 20, 25, 42, 51]

    def test_header_fields(self, example_alto):
        buf = io.BytesIO()
        alto.write_alto(example_alto, buf)
        raw = buf.getvalue()
        assert raw[:4] == b"ALTO" and int.from_bytes(raw[4:8], "little") == 1
        assert raw[8] == 64 and raw[9] == 3
        assert [int.from_bytes(raw[12 + 8 * i: 20 + 8 * i], "little") for i in range(3)] == [4, 8, 2]
        assert int.from_bytes(raw[36:44], "little") == 6
        assert len(raw) == 44 + example_alto.layout.total_bits + 6 * 8 + 6 * 8

    def test_bad_magic(self):
        with pytest.raises(alto.AltoFormatError, match="magic"):
            alto.read_alto(io.BytesIO(b"NOPE" + b"\0" * 64))

    def test_bad_version(self, example_alto):
        buf = io.BytesIO()
        alto.write_alto(example_alto, buf)
        raw = bytearray(buf.getvalue())
        raw[4] = 9
        with pytest.raises(alto.AltoFormatError, match="version"):
            alto.read_alto(io.BytesIO(bytes(raw)))

    def test_bad_width_and_schedule(self, example_alto):
        buf = io.BytesIO()
        alto.write_alto(example_alto, buf)
        raw = bytearray(buf.getvalue())
        w = bytearray(raw)
        w[8] = 128
        with pytest.raises(alto.AltoFormatError, match="width"):
            alto.read_alto(io.BytesIO(bytes(w)))
        s = bytearray(raw)
        s[44] = 7  # schedule names a mode that does not exist
        with pytest.raises(alto.AltoFormatError, match="schedule"):
            alto.read_alto(io.BytesIO(bytes(s)))
        with pytest.raises(alto.AltoFormatError, match="truncated"):
            alto.read_alto(io.BytesIO(bytes(raw[:20])))

    def test_truncated(self, example_alto):
        buf = io.BytesIO()
        alto.write_alto(example_alto, buf)
        with pytest.raises(alto.AltoFormatError, match="truncated"):
            alto.read_alto(io.BytesIO(buf.getvalue()[:-10]))

    def test_unsorted_positions_rejected(self, example_alto):
        buf = io.BytesIO()
        alto.write_alto(example_alto, buf)
        raw = bytearray(buf.getvalue())
        off = 4 + 8 + 24 + 8 + 6
        raw[off:off + 8], raw[off + 8:off + 16] = raw[off + 8:off + 16], raw[off:off + 8]
        with pytest.raises(alto.AltoFormatError, match="invariant"):
            alto.read_alto(io.BytesIO(bytes(raw)))

    def test_wide_roundtrip(self, tmp_path):
        rng = np.random.default_rng(3)
        dims = (2**18, 2**17, 2**17, 2**17)
        coo = alto.CooTensor(dims, *random_sparse(rng, dims, 64))
        t = alto.AltoTensor.from_coo(coo)
        path = tmp_path / "wide.alto"
        alto.write_alto(t, str(path))
        back = alto.read_alto(str(path))
        assert back.to_coo() == coo
        assert np.array_equal(back.positions, t.positions)

    def test_large_file_chunks(self, tmp_path, monkeypatch):
        # force many pinned chunks through the double-buffered loader
        from paper_2403_06348_b200 import io as aio
        monkeypatch.setattr(aio, "_CHUNK_BYTES", 1 << 12)
        rng = np.random.default_rng(5)
        coo = alto.CooTensor((300, 200, 100), *random_sparse(rng, (300, 200, 100), 5000))
        t = alto.AltoTensor.from_coo(coo)
        path = tmp_path / "big.alto"
        alto.write_alto(t, str(path))
        back = alto.read_alto(str(path))
        assert np.array_equal(back.positions, t.positions)
        assert np.array_equal(back.values, t.values)


class TestTextRoundtrip:
    def test_parse_emit_identity(self):
        rng = np.random.default_rng(4)
        for _ in range(5):
            coo = alto.CooTensor((6, 3, 9), *random_sparse(rng, (6, 3, 9), 25))
            buf = io.StringIO()
            alto.write_frostt(coo, buf)
            assert alto.parse_frostt(io.StringIO(buf.getvalue()), dims=coo.shape.dims) == coo


def test_huge_nnz_header_is_a_format_error_not_an_allocation(example_alto):
    """A header announcing far more nonzeros than the stream holds raises the
    reference's 'truncated payload' before any device allocation
    (pkg/src/alto/tensor.py:400-403)."""
    import struct

    buf = io.BytesIO()
    alto.write_alto(example_alto, buf)
    raw = bytearray(buf.getvalue())
    ndim = example_alto.ndim
    off = 4 + 8 + 8 * ndim  # magic, <IBBH>, dims
    raw[off:off + 8] = struct.pack("<Q", 1 << 45)
    with pytest.raises(alto.AltoFormatError, match="truncated payload"):
        alto.read_alto(io.BytesIO(bytes(raw)))
