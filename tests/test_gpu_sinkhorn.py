"""Sinkhorn / IBP baselines on the GPU vs the reference's golden vectors (sinkhorn.py)."""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import device_cost, golden_names, load, rel_err

pytestmark = pytest.mark.gpu

SINKHORN = golden_names("sinkhorn_")


@pytest.mark.parametrize("name", SINKHORN)
def test_sinkhorn_vs_reference(name):
    from paper_2511_11359_b200 import sinkhorn as SK
    d = load(name)
    k = device_cost(d)
    r, c = d["r"], d["c"]
    for eta, tol, mi in ((0.05, 1e-9, 10000), (0.01, 1e-8, 20000), (0.01, 1e-12, 7)):
        tag = f"eta{eta}_mi{mi}"
        pot = SK.sinkhorn_solve(k, r, c, eta, tol=tol, max_iter=mi)
        info = d[f"{tag}_info"]
        assert pot.converged == bool(info[0]) and pot.sweeps == int(info[1]), tag
        assert abs(pot.col_gap - info[2]) <= 1e-11 + 1e-6 * info[2]
        assert rel_err(pot.phi, d[f"{tag}_phi"]) <= 1e-10 and rel_err(pot.psi, d[f"{tag}_psi"]) <= 1e-10
        assert abs(SK.eot_dual_value(pot, k, r, c) - float(d[f"{tag}_dual"])) <= 1e-11
        assert rel_err(SK.sinkhorn_column_marginal(pot, k), d[f"{tag}_col"]) <= 1e-10


def test_ibp_vs_reference():
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200 import sinkhorn as SK
    d = load("ibp_grid5x5_m3")
    g = core.GridKernel(5, 5, 2)
    margs = [core.Histogram(h) for h in d["margs"]]
    for eta, tol, mi in ((0.05, 1e-9, 5000), (0.02, 1e-12, 9)):
        tag = f"eta{eta}_mi{mi}"
        res = SK.ibp_barycenter(g, margs, d["w"], eta, tol=tol, max_iter=mi)
        info = d[f"{tag}_info"]
        assert res.converged == bool(info[0]) and res.sweeps == int(info[1])
        assert rel_err(res.barycenter.weights, d[f"{tag}_bary"]) <= 1e-10
        assert rel_err(res.phis, d[f"{tag}_phis"]) <= 1e-10 and rel_err(res.psis, d[f"{tag}_psis"]) <= 1e-10


def test_sinkhorn_errors_like_reference():
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200 import sinkhorn as SK
    k = core.GridKernel(3, 3, 1)
    with pytest.raises(ValueError):
        SK.sinkhorn_solve(k, np.full(9, 1 / 9), np.full(9, 1 / 9), 0.0)
    r = np.full(9, 1 / 8)
    r[0] = 0.0
    with pytest.raises(ValueError):
        SK.sinkhorn_solve(k, r, np.full(9, 1 / 9), 0.1)


@pytest.mark.parametrize("eta", [5e-2, 5e-4])
def test_grid_separable_sinkhorn_and_ibp_match_dense(eta):
    """GridKernel Sinkhorn / IBP sweeps run as separable LSE convolutions (tensor-core GEMMs at
    eta = 5e-2, exact log-domain convolutions at eta = 5e-4 where exp(-C/eta) would underflow);
    the same cost as an ExplicitKernel takes the dense n^2 sweeps."""
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200 import sinkhorn as SK
    H, W = 24, 19
    n = H * W
    rng = np.random.default_rng(int(1 / eta))
    g = core.GridKernel(H, W, 2)
    e = core.ExplicitKernel(g.materialize(n))
    r = O.normalized_hist(rng.random(n) + 0.1)
    c = O.normalized_hist(rng.random(n) + 0.1)
    ps = SK.sinkhorn_solve(g, r, c, eta, tol=1e-9, max_iter=400)
    pd = SK.sinkhorn_solve(e, r, c, eta, tol=1e-9, max_iter=400)
    assert ps.sweeps == pd.sweeps and ps.converged == pd.converged
    assert rel_err(ps.phi, pd.phi) <= 1e-9 and rel_err(ps.psi, pd.psi) <= 1e-9
    margs = [O.normalized_hist(rng.random(n) + 0.1) for _ in range(3)]
    bs = SK.ibp_barycenter(g, margs, [0.2, 0.3, 0.5], eta, tol=1e-9, max_iter=200)
    bd = SK.ibp_barycenter(e, margs, [0.2, 0.3, 0.5], eta, tol=1e-9, max_iter=200)
    assert bs.sweeps == bd.sweeps
    assert rel_err(bs.barycenter.weights, bd.barycenter.weights) <= 1e-9


def test_dense_plans_match_numpy_from_potentials():
    """sinkhorn_plan_dense / ibp_plan_dense (sinkhorn.py:153-159, 231-236) through the device
    plan kernel agree with exp((phi + psi - C) / eta) computed on the host."""
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200 import sinkhorn as sk
    rng = np.random.default_rng(12)
    n = 90
    Cm = rng.random((n, n))
    k = core.ExplicitKernel(Cm)
    r = core.Histogram.normalized(rng.random(n) + 0.1)
    c = core.Histogram.normalized(rng.random(n) + 0.1)
    pot = sk.sinkhorn_solve(k, r, c, 0.05, tol=1e-10, max_iter=5000)
    Cn = Cm / Cm.max()
    ref = np.exp((pot.phi[:, None] + pot.psi[None, :] - Cn) / pot.eta)
    assert rel_err(sk.sinkhorn_plan_dense(pot, k), ref / ref.sum()) <= 1e-12
    res = sk.ibp_barycenter(k, [r, c], np.array([0.4, 0.6]), 0.05, tol=1e-9, max_iter=2000)
    for q in range(2):
        ref = np.exp((res.phis[q][:, None] + res.psis[q][None, :] - Cn) / res.eta)
        assert rel_err(sk.ibp_plan_dense(res, k, q), ref) <= 1e-12
