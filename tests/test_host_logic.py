"""Host-side logic of the product package (no GPU needed): layout schedule,
scalar codec, span tables, statistics, strategy rules, configs, model, and
the R x R algebra. Mirrors the reference's unit tests for these pieces
(pkg/tests/test_encoding.py, test_kernels.py::TestSelectStrategy,
test_model.py, test_cpd_*.py config validation)."""

import itertools
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2403_06348_b200 as alto
from conftest import golden
from paper_2403_06348_b200 import _native as nat
from paper_2403_06348_b200.cpd import (
    CpAlsConfig,
    CpAprConfig,
    KruskalModel,
    gram,
    hadamard_chain,
    init_factors,
    kkt_violation,
    select_krp_memory_mode,
    solve_pseudo,
)
from paper_2403_06348_b200.encoding import (
    TensorShape,
    UnsupportedShapeError,
    build_layout,
    delinearize,
    layout_from_schedule,
    lexicographic_layout,
    linearize,
    word_spans,
)
from paper_2403_06348_b200.kernels import REUSE_THRESHOLD, Strategy, flops_per_nonzero, select_strategy
from paper_2403_06348_b200.partition import balanced_bounds
from paper_2403_06348_b200.tensor import TensorStats, classify_reuse


class TestLayout:
    def test_worked_schedule(self):
        lay = build_layout((4, 8, 2))
        assert [m for m, _ in reversed(lay.schedule)] == [1, 1, 0, 1, 0, 2]
        for c, p in [((0, 0, 0), 0), ((3, 7, 1), 63), ((1, 0, 0), 2), ((0, 3, 0), 20),
                     ((2, 2, 1), 25), ((1, 6, 1), 51)]:
            assert linearize(lay, c) == p
            assert delinearize(lay, p) == c

    def test_golden_schedules(self):
        g = golden("layouts")
        i = 0
        while f"dims{i}" in g:
            dims = tuple(int(x) for x in g[f"dims{i}"])
            lay = build_layout(dims)
            assert lay.schedule == tuple(tuple(int(v) for v in p) for p in g[f"sched{i}"])
            for pt, want in zip(g[f"pts{i}"], g[f"lin{i}"]):
                assert linearize(lay, pt) == int(want)
            i += 1

    def test_baseline_key_widths(self):
        # c3 needs 71 index bits: 128-bit keys, exactly like the reference
        assert build_layout((2_000_000, 2_000_000, 2_000_000, 168)).total_bits == 71
        assert build_layout((2_000_000, 2_000_000, 2_000_000, 168)).word_bits == 128
        assert build_layout((10_000_000, 10_000_000, 1_000_000, 100_000, 1000)).total_bits == 95
        assert build_layout((12000, 9000, 28000)).word_bits == 64

    def test_tie_break_and_degenerate(self):
        assert build_layout((4, 4)).schedule == ((0, 0), (1, 0), (0, 1), (1, 1))
        lay = build_layout((1, 1, 1))
        assert lay.total_bits == 0 and linearize(lay, (0, 0, 0)) == 0

    def test_errors(self):
        with pytest.raises(ValueError):
            TensorShape(())
        with pytest.raises(ValueError):
            TensorShape((4, 0))
        with pytest.raises(UnsupportedShapeError):
            TensorShape((2**30,) * 5)
        lay = build_layout((4, 8, 2))
        with pytest.raises(IndexError):
            linearize(lay, (4, 0, 0))
        with pytest.raises(ValueError):
            linearize(lay, (0, 0))
        with pytest.raises(ValueError):
            layout_from_schedule((4, 4), [(0, 1), (0, 0), (1, 0), (1, 1)])

    def test_lexicographic_layout_orders_like_tuples(self):
        dims = (3, 5, 2)
        lay = lexicographic_layout(dims)
        pts = list(itertools.product(*(range(d) for d in dims)))
        keys = [linearize(lay, p) for p in pts]
        assert keys == sorted(keys)

    def test_word_spans_split_at_word_edge(self):
        lay = build_layout((2**20,) * 6)
        assert lay.word_bits == 128
        for parts in word_spans(lay):
            for src, bit, ln, word in parts:
                assert 0 <= bit and bit + ln <= 64 and word in (0, 1)
            assert sum(p[2] for p in parts) == 20

    def test_layout_struct_packing(self):
        lay = build_layout((12000, 9000, 28000))
        s = nat.layout_struct(lay)
        assert s.nmodes == 3 and s.word_bits == 64 and s.total_bits == 43
        assert s.span_off[3] == s.nspans
        # rebuild keys from the packed table for random points
        rng = np.random.default_rng(0)
        for _ in range(50):
            pt = [int(rng.integers(0, d)) for d in lay.shape.dims]
            key = 0
            for n in range(3):
                for k in range(s.span_off[n], s.span_off[n + 1]):
                    key |= ((pt[n] >> s.span_src[k]) & ((1 << s.span_len[k]) - 1)) << (
                        s.span_bit[k] + 64 * s.span_word[k])
            assert key == linearize(lay, pt)

    @settings(max_examples=200, deadline=None)
    @given(st.data())
    def test_roundtrip_property(self, data):
        ndim = data.draw(st.integers(1, 6))
        dims = tuple(data.draw(st.integers(1, 2**20)) for _ in range(ndim))
        lay = build_layout(dims)
        c = tuple(data.draw(st.integers(0, d - 1)) for d in dims)
        assert delinearize(lay, linearize(lay, c)) == c

    def test_storage_formulas(self):
        assert alto.alto_metadata_bits((4, 8, 2)) == 6
        assert alto.sfc_metadata_bits((4, 8, 2)) == 9
        assert alto.coo_compression_ratio((4, 8, 2), 8) == Fraction(3)


class TestStatsAndStrategy:
    def test_reuse_classes(self):
        assert classify_reuse(4.9) == "limited"
        assert classify_reuse(5.0) == "medium"
        assert classify_reuse(8.0) == "medium"
        assert classify_reuse(8.1) == "high"

    def test_select_strategy_rules(self):
        s = TensorStats.from_shape_nnz((10, 10, 10), 500)
        assert select_strategy(s, 0, 1).strategy is Strategy.SEQUENTIAL
        lo = TensorStats.from_shape_nnz((10, 39, 39), 39)
        at = TensorStats.from_shape_nnz((10, 40, 40), 40)
        hi = TensorStats.from_shape_nnz((10, 41, 41), 41)
        assert select_strategy(lo, 0, 4).strategy is Strategy.OUTPUT_ORIENTED
        assert select_strategy(at, 0, 4).strategy is Strategy.OUTPUT_ORIENTED
        assert select_strategy(hi, 0, 4).strategy is Strategy.RECURSIVE
        c = select_strategy(hi, 0, 4, buffer_bytes=10_000, temp_budget_bytes=9_999)
        assert c.strategy is Strategy.OUTPUT_ORIENTED and "budget" in c.reason
        assert REUSE_THRESHOLD == 4.0

    def test_choice_json_matches_reference_schema(self):
        s = TensorStats.from_shape_nnz((10, 41, 41), 41)
        d = select_strategy(s, 0, 4).to_json_dict()
        assert set(d) == {"strategy", "mode", "fiber_reuse", "buffer_bytes", "temp_budget_bytes", "reason"}

    def test_flops(self):
        assert flops_per_nonzero(3, 16) == 2 * 16 * 2 + 16
        assert flops_per_nonzero(5, 1) == 9

    def test_memory_mode(self):
        assert select_krp_memory_mode(TensorStats.from_shape_nnz((22500, 22500, 23_800_000), 28_400_000),
                                      16, 105 * 2**20) == "pre"
        assert select_krp_memory_mode(TensorStats.from_shape_nnz((6000, 5700, 244_300, 1200), 54_200_000),
                                      16, 105 * 2**20) == "otf"
        assert select_krp_memory_mode(TensorStats.from_shape_nnz((5, 4, 3), 10), 16, 105 * 2**20) == "otf"

    @settings(max_examples=200, deadline=None)
    @given(st.integers(1, 10_000), st.integers(1, 64))
    def test_balanced_bounds(self, count, parts):
        parts = min(parts, count)
        sizes = np.diff(balanced_bounds(count, parts))
        assert sizes.sum() == count and sizes.max() - sizes.min() <= 1 and sizes.min() >= 1
        base, extra = divmod(count, parts)
        assert (sizes[:extra] == base + 1).all()


class TestConfigsAndModel:
    def test_config_validation(self):
        with pytest.raises(ValueError):
            CpAlsConfig(rank=0)
        with pytest.raises(ValueError):
            CpAlsConfig(max_iters=-1)
        with pytest.raises(ValueError):
            CpAlsConfig(fit_tol=0.0)
        with pytest.raises(ValueError):
            CpAprConfig(max_inner=0)
        with pytest.raises(ValueError):
            CpAprConfig(tau=0.0)
        with pytest.raises(ValueError):
            CpAprConfig(memory_mode="cache")

    def test_init_factors_pinned(self):
        g = golden("drivers")
        m = init_factors((4, 8, 2), 2, seed=42)
        for n, f in enumerate(m.factors):
            assert np.array_equal(f, g[f"init42_factor{n}"])
        assert np.array_equal(m.weights, np.ones(2))

    def test_model_basics(self):
        rng = np.random.default_rng(3)
        m = KruskalModel(np.array([2.0, 3.0]), [rng.random((d, 2)) for d in (3, 4, 5)])
        dense = m.to_dense()
        assert np.isclose(m.norm_squared(), (dense**2).sum(), rtol=1e-12)
        coords = np.array([[0, 1, 2], [2, 3, 4]])
        assert np.allclose(m.values_at(coords), dense[tuple(coords.T)], rtol=1e-12)
        n = m.normalized(1)
        assert np.allclose([f.sum(axis=0) for f in n.factors], 1.0)
        back = KruskalModel.from_json_dict(m.to_json_dict())
        assert np.array_equal(back.weights, m.weights)

    def test_linalg(self):
        rng = np.random.default_rng(4)
        a = rng.random((7, 3))
        assert np.allclose(gram(a), a.T @ a)
        gs = [gram(rng.random((5, 3))) for _ in range(3)]
        assert np.allclose(hadamard_chain(gs, skip=1), gs[0] * gs[2])
        v = gs[0] * gs[2]
        mat = rng.random((6, 3))
        assert np.allclose(solve_pseudo(mat, v), mat @ np.linalg.pinv(v), rtol=1e-8)
        sing = np.outer([1.0, 2.0, 3.0], [1.0, 2.0, 3.0])
        assert np.allclose(solve_pseudo(mat, sing), mat @ np.linalg.pinv(sing), rtol=1e-8)

    def test_kkt(self):
        rng = np.random.default_rng(6)
        b = rng.random((4, 3))
        phi = rng.random((4, 3)) * 2
        naive = max(abs(min(b[i, r], 1 - phi[i, r])) for i in range(4) for r in range(3))
        assert kkt_violation(b, phi) == pytest.approx(naive, rel=1e-15)
        assert kkt_violation(b, np.ones((4, 3))) == 0.0

    def test_padded_ld(self):
        assert [nat.padded_ld(r) for r in (1, 2, 3, 4, 5, 10, 16, 32)] == [4, 4, 4, 4, 8, 16, 16, 32]


def test_public_names_cover_reference_hot_path():
    names = {
        "AltoTensor", "CooTensor", "TensorShape", "AltoLayout", "build_layout", "linearize",
        "delinearize", "make_segments", "make_mode_ordered_view", "Segment", "SegmentSet",
        "ModeOrderedView", "mttkrp", "mttkrp_sequential", "mttkrp_recursive", "mttkrp_output_oriented",
        "select_strategy", "Strategy", "StrategyChoice", "cp_als", "cp_apr_mu", "CpAlsConfig",
        "CpAprConfig", "CpAlsResult", "CpAprResult", "KruskalModel", "init_factors", "phi_kernel",
        "precompute_krp_rows", "kkt_violation", "poisson_loglik", "select_krp_memory_mode",
        "NumericalError", "TensorStats", "compute_stats", "UnsupportedShapeError",
    }
    assert names <= set(alto.__all__)
    for n in names:
        assert hasattr(alto, n)
