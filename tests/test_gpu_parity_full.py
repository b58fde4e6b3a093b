"""Parity at BASELINE scale on the tensors bench.py times (see parity_full.py):
keys / order / segments bit-exact, MTTKRP and driver traces within 1e-9 of
the CPU oracle, CP-APR inner iteration counts identical."""

import pytest

import parity_full as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c3_keys", "c3_shard", "c5_shard"])
def test_full_size_parity(name):
    rep = P.run(name)
    bad = P.failures(rep)
    assert not bad, (bad, rep)
