"""Regression tests for round-1 review findings (needs a B200).

* An evaluation sweep whose row shifts are far off (rows flagged and recomputed by the exact
  fixup) must still give the reference's _plan_stats: the fixup recomputes the row's
  sum e*C and sum e*x with the new shift, not only S (dxg.py:282-310, 412-417).
* leanot_dxg_eval at eta > 0 is idempotent (the row LSEs no longer overwrite the sweep's
  row minima they are shifted by; dxg.py:335-342).
* solve() with a row-restricted stored cost and n <= dense_cap does not materialize the
  dense plan from rows the kernel does not hold (dxg.py:467-471); materialize_plan raises.
"""

import numpy as np
import pytest

import leanot_oracle as O

pytestmark = pytest.mark.gpu


def _inst(n, seed):
    from paper_2511_11359_b200 import core
    rng = np.random.default_rng(seed)
    C = rng.random((n, n))
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    return core.ExplicitKernel(C), O.DenseCost(C), r, c, rng


@pytest.mark.parametrize("eta", [0.0, 1e-3])
def test_eval_sweep_with_fixup_rows_matches_oracle(eta):
    import torch
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n = 700
    k, cost, r, c, rng = _inst(n, 21)
    prm = dxg.params_tuned(eta).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 3.0, n))
    b -= b.max()
    eng = DxgEngine(k, r, c, prm)
    eng.load_state(delta, b, 30.0, 0.1, 30)       # row shifts from the row maxima at a = 30
    a2 = 2500.0
    eng.scal[0] = a2                                # every row's shift is now off by ~1e3
    eng.sweep(evaluate=True)
    torch.cuda.synchronize()
    assert eng.flags[0].item() == 0                 # fixup list consumed
    primal, dual, infeas = eng.evaluate()
    rp, rd, ri, rcol = O.evaluate(O.Iterate(delta, a2, b, 0.1, 30), cost, r, c, eta)
    assert abs(primal - rp) <= 1e-11 * max(1.0, abs(rp))
    assert abs(dual - rd) <= 1e-11 * max(1.0, abs(rd))
    assert abs(infeas - ri) <= 1e-11


def test_eval_eta_positive_is_idempotent():
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n = 2000
    k, cost, r, c, rng = _inst(n, 5)
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    eng = DxgEngine(k, r, c, prm)
    eng.load_state(rng.uniform(-1, 1, n), -np.abs(rng.normal(0, 1, n)), 20.0, 0.02, 20)
    eng.sweep(evaluate=True)
    first = eng.evaluate()
    second = eng.evaluate()
    assert first == second


def test_solve_with_row_restricted_kernel_skips_dense_rounding():
    from paper_2511_11359_b200 import core, dxg
    n = 512
    k = core.HashKernel(n, seed=2, rows=(0, 256))
    rng = np.random.default_rng(2)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-3, max_iter=50), dense_cap=4096)
    assert sol.iterations == 50
    assert getattr(sol, "rounded_plan", None) is None
    with pytest.raises(ValueError):
        dxg.materialize_plan(sol.state.weights, k, r)
