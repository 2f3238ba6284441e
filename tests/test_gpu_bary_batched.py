"""Dense barycenter sweeps with two marginals per read of C (needs a B200).

Plain dense barycenter sweeps run pass A and pass B on K = 4 weight sets {b_k, b_bar_k,
b_k+1, b_bar_k+1} per launch (leanot_bary.cu), so C is read m (not 2m) times per iteration;
an odd m leaves one single-marginal launch.  Checked against the oracle's dxgb_step
(barycenter.py:108-151, pinned to the reference by tests/golden/bary_*) from injected states,
for stored and on-the-fly costs, m = 3 (one pair + one single) and m = 4, and against the
one-marginal-per-pass launches (LEANOT_BARY_BATCH=0).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


def _inst(kind, m, seed):
    from paper_2511_11359_b200 import core
    rng = np.random.default_rng(seed)
    if kind == "stored":
        n = 600
        Cm = rng.random((n, n))
        k, cost = core.ExplicitKernel(Cm), O.DenseCost(Cm)
    else:
        n = 500
        f = rng.random((n, 2))
        k, cost = core.ColorKernel(f, 2), O.PointCost(f, 2)
    margs = [O.normalized_hist(rng.random(n) + 0.05) for _ in range(m)]
    w = rng.random(m) + 0.2
    w /= w.sum()
    deltas = rng.uniform(-0.5, 0.5, (m, n))
    bs = -np.abs(rng.normal(0, 1.5, (m, n)))
    return k, cost, margs, w, deltas, bs


@pytest.mark.parametrize("kind", ["stored", "points"])
@pytest.mark.parametrize("m", [3, 4])
def test_batched_dense_bary_step_matches_oracle(kind, m):
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    k, cost, margs, w, deltas, bs = _inst(kind, m, 10 * m + (kind == "points"))
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    st = B.BarycenterState(deltas.copy(), bs.copy(), 9.0, 0.01, 9, w, prm.eta)
    nxt = B.dxgb_step(st, k, [core.Histogram(h) for h in margs], prm)
    ref = O.bary_step(O.BaryIterate(deltas.copy(), bs.copy(), 9.0, 0.01, 9, w, prm.eta), cost, margs,
                      O.params_tuned(1e-2, tau_mu=0.05))
    assert rel_err(nxt.deltas, ref.deltas) <= 1e-10
    assert rel_err(nxt.bs, ref.bs) <= 1e-10
    assert (nxt.a, nxt.s, nxt.t) == (ref.a, ref.s, ref.t)


def test_batched_matches_one_marginal_per_pass(monkeypatch):
    import torch
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    k, cost, margs, w, deltas, bs = _inst("stored", 5, 3)
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    out = []
    for batch in ("1", "0"):
        monkeypatch.setenv("LEANOT_BARY_BATCH", batch)
        eng = B.BaryEngine(k, [core.Histogram(h) for h in margs], w, prm)
        eng.load_state(deltas, bs, 9.0, 0.01, 9)
        for _ in range(6):
            eng.sweep()
            eng.update()
        torch.cuda.synchronize()
        out.append((eng.col.cpu().numpy().copy(), eng.delta.cpu().numpy().copy()))
    assert rel_err(out[0][0], out[1][0]) <= 1e-12
    assert rel_err(out[0][1], out[1][1]) <= 1e-11


def test_batched_evaluation_sweep_matches_oracle():
    """Evaluation sweeps (one marginal per pass A, pairs in pass B) after plain iterations: the
    pair pass B must see the current (a, a_bar), not the last plain sweep's copy."""
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    k, cost, margs, w, deltas, bs = _inst("stored", 4, 21)
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    eng = B.BaryEngine(k, [core.Histogram(h) for h in margs], w, prm)
    eng.load_state(deltas, bs, 9.0, 0.01, 9)
    for _ in range(3):
        eng.sweep()
        eng.update()
    d2, b2, a2, s2, t2 = eng.read_state()
    eng.sweep(evaluate=True)
    primal, dual, infeas = eng.evaluate()
    ref = O.bary_evaluate(O.BaryIterate(d2, b2, a2, s2, t2, w, prm.eta), cost, margs)
    assert abs(primal - ref[0]) <= 1e-10 * max(1.0, abs(ref[0]))
    assert abs(dual - ref[1]) <= 1e-10 * max(1.0, abs(ref[1]))
    assert rel_err(np.asarray(infeas), np.asarray(ref[2])) <= 1e-9
