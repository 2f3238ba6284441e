"""Edge cases of the solver boundary on the GPU vs the oracle (needs a B200).

Tiny and odd sizes (n = 1, 2, 3, 5, 1023, 1025, 4097: the row-owner / persistent / launch
paths and their boundaries), sparse marginals (zeros in r and, with alpha > 0, in c),
and every error path a user can hit (ValueError as the reference, dxg.py:431-434).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 5, 1023, 1025, 4097])
def test_tiny_and_boundary_sizes_track_oracle(n):
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(n)
    Cm = rng.random((n, n))
    r = O.normalized_hist(rng.random(n) + 0.1)
    c = O.normalized_hist(rng.random(n) + 0.1)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    sol = dxg.solve(core.ExplicitKernel(Cm, cap=None), r, c, prm, dxg.Termination(eps=1e-12, max_iter=60),
                    log_stride=25, dense_cap=0)
    it, conv, iters, traj, col = O.solve(O.DenseCost(Cm), r, c, O.params_tuned(0.0, tau_mu=0.05), eps=1e-12,
                                          max_iter=60)
    assert sol.iterations == iters and sol.converged == conv     # n = 1 converges at the first log point
    # delta lives in [-beta, beta] and b is O(a): compare on those scales (at n = 1 the reference's
    # delta is exactly 0 while the device's is the rounding of 1 - sum_i p_ij, ~1e-16)
    assert np.max(np.abs(sol.state.mu.delta - it.delta)) <= 1e-10 * max(1.0, np.max(np.abs(it.delta)))
    assert np.max(np.abs(sol.state.weights.b - it.b)) <= 1e-10 * max(1.0, np.max(np.abs(it.b)))
    assert abs(sol.final.primal - traj[-1][1]) <= 1e-9 * max(1.0, abs(traj[-1][1]))


def test_sparse_marginals_with_alpha():
    """Zeros in r (rows with no mass) and in c (allowed because alpha > 0, dxg.py:432)."""
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(4)
    n = 300
    Cm = rng.random((n, n))
    rw = rng.random(n)
    rw[rng.choice(n, 60, replace=False)] = 0.0
    cw = rng.random(n)
    cw[rng.choice(n, 40, replace=False)] = 0.0
    r, c = O.normalized_hist(rw), O.normalized_hist(cw)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    sol = dxg.solve(core.ExplicitKernel(Cm), r, c, prm, dxg.Termination(eps=1e-12, max_iter=75), dense_cap=0)
    it, conv, iters, traj, col = O.solve(O.DenseCost(Cm), r, c, O.params_tuned(0.0, tau_mu=0.05), eps=1e-12,
                                          max_iter=75)
    assert sol.iterations == iters
    assert rel_err(sol.state.mu.delta, it.delta) <= 1e-10
    assert rel_err(sol.state.weights.b, it.b) <= 1e-10


def test_error_paths_raise_value_error():
    from paper_2511_11359_b200 import core, dxg
    n = 8
    k = core.ExplicitKernel(np.ones((n, n)))
    r = np.full(n, 1.0 / n)
    c = np.full(n, 1.0 / n)
    c0 = c.copy()
    c0[0], c0[1] = 0.0, 2.0 / n
    with pytest.raises(ValueError):
        dxg.solve(k, r, np.full(n + 1, 1.0 / (n + 1)), dxg.params_tuned(0.0))      # size mismatch
    with pytest.raises(ValueError):
        dxg.solve(k, r, c0, dxg.params_tuned(0.0).with_overrides(alpha=0.0))      # alpha = 0, c not full support
    with pytest.raises(ValueError):
        core.ExplicitKernel(-np.ones((n, n)))                                      # negative cost
    with pytest.raises(ValueError):
        core.ExplicitKernel(np.ones((n, n + 1)))                                   # not square
    with pytest.raises(ValueError):
        dxg.DxgParams(eta=-1.0, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.01)
    with pytest.raises(ValueError):
        core.Histogram(np.array([0.5, 0.6]))                                       # does not sum to 1
