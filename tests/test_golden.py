"""The oracle reproduces the committed golden fixtures (tests/golden/make_golden.py)
bit-for-bit: guards the checker itself against regressions."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden  # noqa: E402


@pytest.mark.parametrize("key", ["c1_n32", "c2_n64", "c3_n16", "c4_n16"])
def test_oracle_reproduces_golden(oracle, key):
    ref = np.load(os.path.join(HERE, "golden", key + ".npz"))
    name, n, steps, kw = make_golden.CASES[key]
    tr, mg, ka, f, cr = make_golden.run(name, n, steps, kw)
    assert np.array_equal(tr, ref["trace"])
    assert np.array_equal(cr, ref["cross"])
    assert np.array_equal(f, ref["fields"])
