"""Device encoder parity: canonicalisation, linearisation, sort order,
segments and mode-ordered views must equal the reference bit for bit
(golden fixtures from the reference itself)."""

import numpy as np
import pytest

import paper_2403_06348_b200 as alto
from conftest import EXAMPLE_COORDS, EXAMPLE_DIMS, EXAMPLE_VALUES, golden, random_cases
from oracle import alto_oracle as orc
from paper_2403_06348_b200.tensor import decode_coords, encode_coords

pytestmark = pytest.mark.gpu


def test_worked_example():
    g = golden("worked")
    coo = alto.CooTensor(EXAMPLE_DIMS, EXAMPLE_COORDS, EXAMPLE_VALUES)
    assert np.array_equal(coo.coords, g["coo_coords"])
    t = alto.AltoTensor.from_coo(coo)
    assert t.position_ints() == [2, 15, 20, 25, 42, 51]
    assert np.array_equal(t.positions, g["positions"])
    assert np.array_equal(t.values, g["values"])
    assert np.array_equal(t.coords, g["coords"])
    segs = alto.make_segments(t, 2)
    assert [(s.pos_first, s.pos_last) for s in segs.segments] == [(2, 20), (25, 51)]
    assert segs.segments[0].intervals == ((0, 3), (0, 3), (0, 1))
    assert segs.segments[1].intervals == ((1, 3), (2, 6), (0, 1))
    one = alto.make_segments(t, 1)
    assert one.segments[0].intervals == ((0, 3), (0, 6), (0, 1))
    assert alto.make_segments(t, 100).num_segments == 6
    v = alto.make_mode_ordered_view(t, 0, 2)
    assert v.coords[:, 0].tolist() == [0, 1, 1, 2, 3, 3]
    assert np.array_equal(v.perm, g["view0_perm"])
    assert v.boundary_rows.tolist() == []
    assert alto.make_mode_ordered_view(t, 0, 2) is v


@pytest.mark.parametrize("case", random_cases())
def test_random_cases_bitexact(case):
    g = golden(case)
    dims = tuple(int(x) for x in g["dims"])
    coo = alto.CooTensor(dims, g["in_coords"], g["in_values"])
    assert np.array_equal(coo.coords, g["coo_coords"])
    assert np.array_equal(coo.values, g["coo_values"])
    t = alto.AltoTensor.from_coo(coo)
    assert np.array_equal(t.positions, g["positions"])
    assert np.array_equal(t.values, g["values"])
    assert np.array_equal(t.coords, g["coords"])
    for L in (1, 2, 4, 7):
        s = alto.make_segments(t, L)
        assert np.array_equal(s.bounds(), g[f"L{L}_bounds"])
        lo = np.asarray([[iv[0] for iv in seg.intervals] for seg in s.segments])
        hi = np.asarray([[iv[1] for iv in seg.intervals] for seg in s.segments])
        assert np.array_equal(lo, g[f"L{L}_lo"]) and np.array_equal(hi, g[f"L{L}_hi"])
        assert [str(x.pos_first) for x in s.segments] == list(g[f"L{L}_pos_first"])
        assert [str(x.pos_last) for x in s.segments] == list(g[f"L{L}_pos_last"])
        for n in range(len(dims)):
            assert np.array_equal(s.boundary_rows[n], g[f"L{L}_boundary{n}"])
    for mode in range(len(dims)):
        for L in (2, 4, 7):
            v = alto.make_mode_ordered_view(t, mode, L)
            assert np.array_equal(v.perm, g[f"view{L}_m{mode}_perm"])
            assert np.array_equal(v.boundary_rows, g[f"view{L}_m{mode}_boundary"])


def test_wide_128bit_keys():
    g = golden("wide128")
    dims = tuple(int(x) for x in g["dims"])
    t = alto.AltoTensor.from_coo(alto.CooTensor(dims, g["in_coords"], g["in_values"]))
    assert t.layout.word_bits == 128 and t.positions.shape == (len(g["values"]), 2)
    assert np.array_equal(t.positions, g["positions"])
    assert np.array_equal(t.values, g["values"])
    assert np.array_equal(t.coords, g["coords"])
    s = alto.make_segments(t, 3)
    assert [str(x.pos_first) for x in s.segments] == list(g["L3_pos_first"])
    ints = t.position_ints()
    assert all(a < b for a, b in zip(ints, ints[1:]))


def test_duplicates_and_zero_drop():
    d = golden("duplicates")
    coo = alto.CooTensor(tuple(d["dims"]), d["in_coords"], d["in_values"])
    assert np.array_equal(coo.coords, d["coo_coords"])
    assert np.array_equal(coo.values, d["coo_values"])  # input-order summation, bitwise


def test_layout_codec_against_oracle():
    g = golden("layouts")
    for i in range(10):
        dims = tuple(int(x) for x in g[f"dims{i}"])
        lay = alto.build_layout(dims)
        keys = encode_coords(lay, g[f"pts{i}"])
        assert np.array_equal(keys, orc.encode(dims, g[f"pts{i}"]))
        assert np.array_equal(decode_coords(lay, keys), g[f"pts{i}"])


def test_errors():
    with pytest.raises(ValueError, match="range"):
        alto.CooTensor((2, 2), [[0, 5]], [1.0])
    with pytest.raises(ValueError, match="finite"):
        alto.CooTensor((2, 2), [[0, 1]], [np.inf])
    with pytest.raises(ValueError):
        alto.AltoTensor.from_coo(alto.CooTensor((2, 2), np.empty((0, 2), dtype=np.int64), []))
    lay = alto.build_layout((4, 8, 2))
    with pytest.raises(IndexError):
        encode_coords(lay, np.array([[4, 0, 0]]))
    with pytest.raises(ValueError, match="increasing"):
        alto.AltoTensor(lay, np.array([15, 2], dtype=np.uint64), [1.0, 2.0])
    lay3 = alto.build_layout((3, 8, 2))  # mode 0 has a hole: index 3
    with pytest.raises(ValueError, match="outside"):
        alto.AltoTensor(lay3, np.array([lay3.masks[0]], dtype=np.uint64), [1.0])
    with pytest.raises(ValueError):
        alto.make_segments(alto.AltoTensor.from_coo(alto.CooTensor((4, 8, 2), EXAMPLE_COORDS, EXAMPLE_VALUES)), 0)


def test_large_sort_and_roundtrip_properties():
    """1M-nonzero c1-shaped tensor: strictly increasing keys, decode round
    trip, and the same key set as the oracle encoder (size-independent
    properties at the BASELINE configs[0] size)."""
    from paper_2403_06348_b200 import synthetic

    cfg = synthetic.CONFIGS["c1"]
    coords, vals = synthetic.generate_numpy(cfg, cfg.nnz, seed=3)
    t = alto.AltoTensor.from_coo(alto.CooTensor(cfg.dims, coords, vals))
    assert t.nnz == cfg.nnz
    keys = t.positions
    assert (keys[1:] > keys[:-1]).all()
    want = np.sort(orc.encode(cfg.dims, coords))
    assert np.array_equal(keys, want)
    order = np.argsort(orc.encode(cfg.dims, coords), kind="stable")
    assert np.array_equal(t.values, vals[order])
    assert np.array_equal(t.coords, coords[order])
