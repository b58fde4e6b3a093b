"""The public mttkrp()'s call memo (memo.CallMemo): a user's CP-ALS loop
calling mttkrp mode by mode gets the memoised sweep's dimension-tree reuse,
decided on the device from a bitwise check of A_k. Every result must match
the oracle's MTTKRP of the factors actually passed (1e-12 relative, the fast
paths' bar) whichever kernel served the call."""

import numpy as np
import pytest

import paper_2403_06348_b200 as alto
from conftest import assert_close_rel, random_sparse
from oracle import alto_oracle as orc

pytestmark = pytest.mark.gpu

DIMS = (300, 200, 400)
R = 16


@pytest.fixture()
def case():
    rng = np.random.default_rng(21)
    coords, vals = random_sparse(rng, DIMS, 60000, kind="positive")
    t = alto.AltoTensor.from_coo(alto.CooTensor(DIMS, coords, vals))
    ocoords, ovals = orc.canonicalize(coords, vals)
    _, svals, scoords = orc.from_coo(DIMS, ocoords, ovals)
    return t, scoords, svals, rng


def _memo(t):
    return t._cache.get(("callmemo", R))


def _check(t, scoords, svals, facs, mode):
    got = alto.mttkrp(t, facs, mode)
    want = orc.mttkrp(scoords, svals, facs, mode, "sequential")
    assert_close_rel(got, want, 1e-12)
    return got


def test_user_cp_als_loop(case):
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for _sweep in range(5):
        for n in range(3):
            m = _check(t, scoords, svals, facs, n)
            # the user's update of mode n (any new values will do)
            g = np.ones((R, R))
            for k in range(3):
                if k != n:
                    g *= facs[k].T @ facs[k]
            facs[n] = m @ np.linalg.pinv(g)
            facs[n] /= np.maximum(np.abs(facs[n]).max(axis=0), 1e-300)
    cm = _memo(t)
    assert cm is not None
    # alternating producer / consumer once the cyclic order is seen
    assert cm.stats["consume"] >= 5 and cm.stats["produce"] >= 5, cm.stats


def test_unchanged_factors(case):
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for _ in range(3):
        for n in range(3):
            _check(t, scoords, svals, facs, n)
    assert _memo(t).stats["consume"] >= 3


def test_changed_ak_forces_the_producer(case):
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for n in (0, 1, 2, 0):
        _check(t, scoords, svals, facs, n)
    cm = _memo(t)
    before = dict(cm.stats)
    # mode 1 would consume mode 0's T (A_2 unchanged); change one bit of A_2
    facs[2] = facs[2].copy()
    facs[2][7, 3] = np.nextafter(facs[2][7, 3], 2.0)
    _check(t, scoords, svals, facs, 1)
    assert cm.stats["produce"] == before["produce"] + 1
    assert cm.stats["consume"] == before["consume"]


def test_non_cyclic_order_bypasses_the_memo(case):
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for n in (0, 2, 1, 1, 0, 0, 2):
        _check(t, scoords, svals, facs, n)
    cm = _memo(t)
    assert cm is None or cm.stats == {"produce": 0, "consume": 0}


def test_non_finite_factor_raises_and_recovers(case):
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for n in (0, 1, 2):
        _check(t, scoords, svals, facs, n)
    bad = [f.copy() for f in facs]
    bad[1][3, 2] = np.inf
    with pytest.raises(ValueError, match="factor 1"):
        alto.mttkrp(t, bad, 0)
    for n in (0, 1, 2, 0, 1):
        _check(t, scoords, svals, facs, n)


def test_env_switch_off(case, monkeypatch):
    monkeypatch.setenv("ALTO_B200_CALL_MEMO", "0")
    t, scoords, svals, rng = case
    facs = [rng.random((d, R)) for d in DIMS]
    for _ in range(2):
        for n in range(3):
            _check(t, scoords, svals, facs, n)
    assert _memo(t) is None
