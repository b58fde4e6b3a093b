"""CpAls / CpApr estimator wrappers: the parameter protocol (CPU) and fits
through the GPU drivers (reference cases: pkg/tests/test_estimators.py)."""

import numpy as np
import pytest

import paper_2403_06348_b200 as alto
from conftest import random_sparse
from paper_2403_06348_b200.estimators import as_alto_tensor


class TestParamProtocol:
    def test_get_set_params(self):
        est = alto.CpAls(rank=4)
        params = est.get_params()
        assert params["rank"] == 4 and params["max_iters"] == 50 and params["exact"] is None
        est.set_params(rank=2, seed=7)
        assert est.rank == 2 and est.seed == 7
        with pytest.raises(ValueError, match="invalid parameter"):
            est.set_params(bogus=1)
        with pytest.raises(TypeError):
            alto.CpApr(bogus=1)

    def test_sklearn_clone_compatible(self):
        sklearn_base = pytest.importorskip("sklearn.base")
        est = alto.CpApr(rank=3, tau=1e-3)
        cloned = sklearn_base.clone(est)
        assert cloned is not est and cloned.get_params() == est.get_params()

    def test_repr_and_signature(self):
        import inspect

        assert "rank=5" in repr(alto.CpAls(rank=5))
        assert "max_outer" in inspect.signature(alto.CpApr).parameters
        assert "max_iters" not in inspect.signature(alto.CpApr).parameters

    def test_unfitted_raises(self):
        with pytest.raises(RuntimeError, match="not fitted"):
            alto.CpAls().score()

    def test_rejects_garbage(self):
        with pytest.raises(TypeError):
            as_alto_tensor(object())


@pytest.fixture(scope="module")
def small_tensor():
    rng = np.random.default_rng(40)
    return alto.CooTensor((5, 4, 3), *random_sparse(rng, (5, 4, 3), 30))


@pytest.fixture(scope="module")
def count_data():
    rng = np.random.default_rng(41)
    return alto.CooTensor((5, 4, 3), *random_sparse(rng, (5, 4, 3), 30, kind="counts"))


@pytest.mark.gpu
class TestFits:
    def test_cp_als_fit_attributes(self, small_tensor):
        est = alto.CpAls(rank=2, max_iters=10, seed=0).fit(small_tensor)
        assert est.model_.rank == 2 and len(est.factors_) == 3 and est.n_iters_ <= 10
        assert est.score() == est.fit_trace_[-1]
        direct = alto.cp_als(alto.AltoTensor.from_coo(small_tensor), alto.CpAlsConfig(rank=2, max_iters=10))
        assert est.fit_trace_ == direct.fit_trace
        assert est.predict(small_tensor.coords).shape == (small_tensor.nnz,)

    def test_cp_als_accepts_dense(self):
        rng = np.random.default_rng(42)
        est = alto.CpAls(rank=1, max_iters=5, seed=0).fit(rng.random((4, 3, 2)))
        assert est.model_.shape == (4, 3, 2)

    def test_cp_apr_fit_attributes(self, count_data):
        est = alto.CpApr(rank=2, max_outer=30, seed=0).fit(count_data)
        assert est.model_.rank == 2 and est.memory_mode_ in ("pre", "otf")
        assert all((f >= 0).all() for f in est.factors_)
        assert np.isfinite(est.score(count_data))
        exact = alto.CpApr(rank=2, max_outer=30, seed=0, exact=True).fit(count_data)
        assert exact.inner_iters_ == est.inner_iters_

    def test_cp_apr_rejects_negative(self, small_tensor):
        with pytest.raises(ValueError, match="negative"):
            alto.CpApr(rank=1, max_outer=2).fit(small_tensor)

    def test_coercion(self, small_tensor):
        t = as_alto_tensor(small_tensor)
        assert t.nnz == small_tensor.nnz and as_alto_tensor(t) is t
