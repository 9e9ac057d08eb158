"""The oracle (CPU restatement, oracle/) reproduces the reference bit-for-bit.

Pins the oracle against outputs of the reference itself (tests/golden/*.npz,
made by tests/golden/make_golden.py from /root/reference).  In the build
container numpy is the same build the goldens came from, so even the
transcendental-derived scalars (rho, epsilon_achieved) must match exactly;
on another host they are compared at 1e-12 relative.
"""

import json

import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, GoldenCase, assert_outcome, golden_names


def _same_numpy(case):
    return case.meta["numpy"] == np.__version__


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_goldens(name):
    case = GoldenCase(name)
    rtol = 0.0 if _same_numpy(case) else TRANS_RTOL
    T, ix = case.table, case.index
    for st in case.steps():
        if st["variant"] == "incremental":
            out = O.decode_step(T, ix, st["h"], st["cfg"], k_max=st["k_max"])
        else:
            out = O.decode_step_batchselect(T, ix, st["h"], st["cfg"], k_max=st["k_max"])
        exp = case.expected(st["i"])
        assert_outcome(out, exp, rtol=rtol, where=f"{name}[{st['i']}]")
        b = O.cluster_bounds(ix, st["h"], slack_mode=st["cfg"].slack_mode)
        if ix.mode != "spherical" or _same_numpy(case):
            assert np.array_equal(b.values, exp["U"]), f"{name}[{st['i']}]: bounds differ"
        else:
            np.testing.assert_allclose(b.values, exp["U"], rtol=1e-12)
        assert b.query_norm == exp["qn"]
        assert b.slack == exp["slack"]


@pytest.mark.parametrize("name", golden_names())
def test_oracle_dense_matches_reference(name):
    case = GoldenCase(name)
    for i, ref in enumerate(case.z["dense"]):
        logits, probs, order = O.dense_logits(case.table, case.z["queries"][i])
        assert np.array_equal(logits, ref)
