"""scikit-learn style estimators over the GPU drivers.

API of pkg/src/alto/estimators.py (``CpAls``, ``CpApr``, ``as_alto_tensor``):
constructor keywords mirror the driver configs and round-trip through
``get_params``/``set_params`` (so ``sklearn.base.clone`` works without this
package importing scikit-learn), fitted state lives in trailing-underscore
attributes, and ``fit`` accepts an ``AltoTensor``, a ``CooTensor`` or a
dense array. Here the parameter list is derived from the config dataclass,
plus ``exact`` (``True`` runs the reference's accumulation order bit for
bit).
"""

from __future__ import annotations

import dataclasses
import inspect

import numpy as np

from .cpd import CpAlsConfig, CpAprConfig, cp_als, cp_apr_mu, poisson_loglik
from .tensor import AltoTensor, CooTensor


def as_alto_tensor(data) -> AltoTensor:
    """AltoTensor | CooTensor | dense array -> AltoTensor (device resident)."""
    if isinstance(data, AltoTensor):
        return data
    if isinstance(data, CooTensor):
        return AltoTensor.from_coo(data)
    arr = np.asarray(data)
    if arr.dtype == object or arr.ndim < 1:
        raise TypeError(f"cannot interpret {type(data).__name__} as a sparse tensor")
    return AltoTensor.from_coo(CooTensor.from_dense(arr))


class _DriverEstimator:
    """Parameters = the config dataclass's fields (+ ``exact``)."""

    _config: type = None
    _driver = None
    _skip_fields: tuple = ()
    # fitted attribute -> attribute path on the driver result
    _outputs: dict = {}

    @classmethod
    def _fields(cls):
        return [f for f in dataclasses.fields(cls._config) if f.name not in cls._skip_fields]

    @classmethod
    def _param_names(cls):
        return [f.name for f in cls._fields()] + ["exact"]

    def __init_subclass__(cls, **kw):
        super().__init_subclass__(**kw)
        params = [inspect.Parameter("self", inspect.Parameter.POSITIONAL_OR_KEYWORD)]
        for f in cls._fields():
            params.append(inspect.Parameter(f.name, inspect.Parameter.KEYWORD_ONLY, default=f.default))
        params.append(inspect.Parameter("exact", inspect.Parameter.KEYWORD_ONLY, default=None))

        def __init__(self, **kwargs):
            _DriverEstimator.__init__(self, **kwargs)

        __init__.__signature__ = inspect.Signature(params)
        cls.__init__ = __init__

    def __init__(self, **params):
        defaults = {f.name: f.default for f in self._fields()}
        defaults["exact"] = None
        unknown = set(params) - set(defaults)
        if unknown:
            raise TypeError(f"{type(self).__name__} got unexpected parameters {sorted(unknown)}")
        for name, default in defaults.items():
            setattr(self, name, params.get(name, default))

    def get_params(self, deep: bool = True) -> dict:
        return {name: getattr(self, name) for name in self._param_names()}

    def set_params(self, **params):
        valid = set(self._param_names())
        for name, value in params.items():
            if name not in valid:
                raise ValueError(f"invalid parameter {name!r} for {type(self).__name__}")
            setattr(self, name, value)
        return self

    def __repr__(self):
        return f"{type(self).__name__}({', '.join(f'{k}={v!r}' for k, v in self.get_params().items())})"

    def _make_config(self):
        return self._config(**{f.name: getattr(self, f.name) for f in self._fields()})

    def fit(self, X, y=None):
        tensor = as_alto_tensor(X)
        result = type(self)._driver(tensor, self._make_config(), exact=self.exact)
        self.result_ = result
        self.model_ = result.model
        self.weights_ = result.model.weights
        self.factors_ = result.model.factors
        for attr, src in self._outputs.items():
            setattr(self, attr, getattr(result, src))
        return self

    def predict(self, coords) -> np.ndarray:
        """Model values at zero-based (M, N) coordinates."""
        self._check_fitted()
        return self.model_.values_at(np.asarray(coords))

    def _check_fitted(self):
        if not hasattr(self, "model_"):
            raise RuntimeError("estimator is not fitted; call fit first")


class CpAls(_DriverEstimator):
    """Least-squares CP (CP-ALS). Fitted: ``weights_``, ``factors_``,
    ``model_``, ``fit_trace_``, ``objective_trace_``, ``n_iters_``,
    ``converged_``, ``strategies_``, ``result_``."""

    _config = CpAlsConfig
    _driver = staticmethod(cp_als)
    _outputs = {"fit_trace_": "fit_trace", "objective_trace_": "objective_trace", "n_iters_": "n_iters",
                "converged_": "converged", "strategies_": "strategies"}

    def score(self, X=None, y=None) -> float:
        """Final fit 1 - |X - model|_F / |X|_F of the training run."""
        self._check_fitted()
        return self.fit_trace_[-1]


class CpApr(_DriverEstimator):
    """Poisson CP (CP-APR, multiplicative updates). Fitted: ``weights_``,
    ``factors_``, ``model_``, ``kkt_trace_``, ``inner_iters_``,
    ``loglik_trace_``, ``n_outer_``, ``converged_``, ``memory_mode_``,
    ``strategies_``, ``result_``."""

    _config = CpAprConfig
    _driver = staticmethod(cp_apr_mu)
    _skip_fields = ("track_inner_loglik",)
    _outputs = {"kkt_trace_": "kkt_trace", "inner_iters_": "inner_iters", "loglik_trace_": "loglik_trace",
                "n_outer_": "n_outer", "converged_": "converged", "memory_mode_": "memory_mode",
                "strategies_": "strategies"}

    def score(self, X, y=None) -> float:
        """Poisson log-likelihood of the fitted model on X."""
        self._check_fitted()
        return poisson_loglik(as_alto_tensor(X), self.model_)


__all__ = ["CpAls", "CpApr", "as_alto_tensor"]
