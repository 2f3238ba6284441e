"""Intrinsic noise floor of the reference algorithm (CPU, oracle only).

Changing nothing but the row-block size (summation order) of the reference's
sweeps shows which regimes amplify rounding noise.  This is what bounds a
meaningful per-iteration parity horizon for ANY re-implementation.
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import load, oracle_cost, params_from, rel_err


def _run(d, scheme, steps, block_rows):
    cost = oracle_cost(d)
    prm = params_from(d[f"{scheme}_params"])
    orig = O.row_blocks
    O.row_blocks = lambda n, _ignored=None, br=block_rows: orig(n, br)
    try:
        it = O.Iterate.zero(cost.n)
        out = []
        for _ in range(steps):
            it = O.step(it, cost, d["r"], d["c"], prm)
            out.append(it.delta.copy())
    finally:
        O.row_blocks = orig
    return out


def test_li_regime_amplifies_summation_order_noise():
    d = load("step_explicit_n200")
    a = _run(d, "li", 40, 128)
    b = _run(d, "li", 40, 16)
    assert rel_err(b[0], a[0]) < 1e-14
    assert rel_err(b[-1], a[-1]) > 1e-10     # the reference alone leaves 1e-10


@pytest.mark.parametrize("scheme", ["tuned_taumu005", "loose"])
def test_non_chaotic_regimes_stay_at_rounding_level(scheme):
    d = load("step_explicit_n200")
    a = _run(d, scheme, 40, 128)
    b = _run(d, scheme, 40, 16)
    assert max(rel_err(x, y) for x, y in zip(b, a)) < 1e-12
