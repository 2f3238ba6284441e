"""Barycenter (Alg. 4) on the GPU vs the reference's golden vectors (barycenter.py)."""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import load, rel_err

pytestmark = pytest.mark.gpu


def _setup():
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    d = load("bary_grid5x5_m3")
    g = core.GridKernel(5, 5, 2)
    prm = dxg.DxgParams(*[float(v) for v in d["params"]])
    margs = [core.Histogram(h) for h in d["margs"]]
    st = B.BarycenterState(d["in_deltas"].copy(), d["in_bs"].copy(), float(d["in_scalars"][0]),
                           float(d["in_scalars"][1]), int(d["in_scalars"][2]), d["w"], prm.eta)
    return B, core, dxg, d, g, prm, margs, st


def test_barycenter_marginal_and_objective():
    B, core, dxg, d, g, prm, margs, st = _setup()
    r = B.barycenter_marginal(st, g)
    assert rel_err(r.weights, d["rmap"]) <= 1e-12
    obj = B.barycenter_objective(st, g, margs)
    assert abs(obj - float(d["objective"])) <= 1e-11 * max(1.0, abs(obj))


def test_dxgb_step_injected_state():
    B, core, dxg, d, g, prm, margs, st = _setup()
    nxt = B.dxgb_step(st, g, margs, prm)
    assert rel_err(nxt.deltas, d["out_deltas"]) <= 1e-10
    assert rel_err(nxt.bs, d["out_bs"]) <= 1e-10
    assert [nxt.a, nxt.s, nxt.t] == d["out_scalars"].tolist()


def test_folded_evaluation_matches_reference():
    B, core, dxg, d, g, prm, margs, st = _setup()
    eng = B.BaryEngine(g, margs, st.w, prm)
    eng.load_state(st.deltas, st.bs, st.a, st.s, st.t)
    eng.sweep(evaluate=True)
    primal, dual, infeas = eng.evaluate()
    assert abs(primal - float(d["eval_primal"])) <= 1e-11
    assert abs(dual - float(d["eval_dual"])) <= 1e-11
    assert rel_err(infeas, d["eval_infeas"]) <= 1e-10


def test_dxgb_solve_same_iterations_and_barycenter():
    B, core, dxg, d, g, prm, margs, st = _setup()
    sol = B.dxgb_solve(g, margs, d["w"], prm, dxg.Termination(eps=5e-3, max_iter=3000), log_stride=25)
    assert sol.converged == bool(d["solve_converged"])
    assert sol.iterations == int(d["solve_iterations"])
    assert rel_err(sol.barycenter.weights, d["solve_bary"]) <= 1e-9
    got = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    ref = d["solve_traj"]
    assert got.shape == ref.shape and np.array_equal(got[:, 0], ref[:, 0])
    assert rel_err(got[:, 1], ref[:, 1]) <= 1e-8 and rel_err(got[:, 2], ref[:, 2]) <= 1e-8
    assert rel_err(sol.state.deltas, d["solve_deltas"]) <= 1e-8
    assert rel_err(sol.per_marginal_infeas, d["solve_infeas"]) <= 1e-7


def test_barycenter_larger_grid_vs_oracle():
    """16x16 grid, m=4, against the oracle restatement (several iterations)."""
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(3)
    n, m = 256, 4
    M = [O.normalized_hist(rng.random(n) + 0.1) for _ in range(m)]
    w = np.array([0.1, 0.2, 0.3, 0.4])
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    oprm = O.params_tuned(1e-2, tau_mu=0.05)
    gk, og = core.GridKernel(16, 16, 2), O.GridCost(16, 16, 2)
    eng = B.BaryEngine(gk, M, w, prm)
    eng.load_state(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, fresh=True)
    ost = O.BaryIterate.zero(n, w, prm.eta)
    for it in range(30):
        eng.sweep()
        eng.update()
        ost = O.bary_step(ost, og, M, oprm)
    deltas, bs, a, s, t = eng.read_state()
    assert rel_err(deltas, ost.deltas) <= 1e-10
    assert rel_err(bs, ost.bs) <= 1e-10
    assert (a, s, t) == (ost.a, ost.s, ost.t)
