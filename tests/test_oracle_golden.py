"""Pin the CPU oracle (oracle/leanot_oracle.py) against the reference's own outputs.

Fixtures in tests/golden were produced by running the reference (`leanot`) in the
build container (oracle/gen_golden.py).  No GPU needed.
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import golden_names, load, oracle_cost, params_from, rel_err

SWEEPS = golden_names("sweep_")
STEPS = golden_names("step_")
SOLVES = golden_names("solve_")


@pytest.mark.parametrize("name", SWEEPS)
def test_sweeps_match_reference(name):
    d = load(name)
    cost = oracle_cost(d)
    r, c = d["r"], d["c"]
    for t in range(3):
        a, b, delta = float(d[f"case{t}_a"]), d[f"case{t}_b"], d[f"case{t}_delta"]
        (col,) = O.column_marginals(cost, r, [(a, b)])
        assert rel_err(col, d[f"case{t}_col"]) <= 1e-14
        cst, col2, ent = O.plan_stats(a, b, cost, r)
        assert abs(cst - float(d[f"case{t}_cost"])) <= 1e-14 * max(1.0, abs(cst))
        assert abs(ent - float(d[f"case{t}_ent"])) <= 1e-13 * max(1.0, abs(ent))
        for key, eta in (("dual0", 0.0), ("dual3", 1e-3), ("dual7", 1e-7)):
            v = O.dual_value(delta, cost, r, c, eta)
            assert abs(v - float(d[f"case{t}_{key}"])) <= 1e-13 * max(1.0, abs(v)), key
    phi, psi = O.recover_potentials(d["case1_delta"], cost, d["r_full"], 1e-2)
    assert rel_err(phi, d["pot_phi"]) <= 1e-13
    assert rel_err(psi, d["pot_psi"]) <= 1e-13


SCHEMES = ["tuned", "tuned_taumu005", "tuned_eta1e-3", "loose", "li"]


@pytest.mark.parametrize("name", STEPS)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_step_matches_reference(name, scheme):
    d = load(name)
    cost = oracle_cost(d)
    prm = params_from(d[f"{scheme}_params"])
    a, s, t = d[f"{scheme}_in_scalars"]
    it = O.Iterate(d[f"{scheme}_in_delta"], float(a), d[f"{scheme}_in_b"], float(s), int(t))
    nxt = O.step(it, cost, d["r"], d["c"], prm)
    assert rel_err(nxt.delta, d[f"{scheme}_out_delta"]) <= 1e-13
    assert rel_err(nxt.b, d[f"{scheme}_out_b"]) <= 1e-13
    assert [nxt.a, nxt.s, nxt.t] == d[f"{scheme}_out_scalars"].tolist()


@pytest.mark.parametrize("name", STEPS)
@pytest.mark.parametrize("scheme", ["tuned_taumu005", "loose", "li", "tuned_eta1e-3"])
def test_short_trajectory_matches_reference(name, scheme):
    d = load(name)
    cost = oracle_cost(d)
    prm = params_from(d[f"{scheme}_params"])
    it = O.Iterate.zero(cost.n)
    for k in range(d[f"{scheme}_traj_delta"].shape[0]):
        it = O.step(it, cost, d["r"], d["c"], prm)
        assert rel_err(it.delta, d[f"{scheme}_traj_delta"][k]) <= 1e-12, k
        assert rel_err(it.b, d[f"{scheme}_traj_b"][k]) <= 1e-12, k


@pytest.mark.parametrize("name", SOLVES)
def test_solve_matches_reference(name):
    d = load(name)
    cost = oracle_cost(d)
    prm = params_from(d["params"])
    eps, max_iter = float(d["term"][0]), int(d["term"][1])
    it, conv, k, traj, col = O.solve(cost, d["r"], d["c"], prm, eps=eps, max_iter=max_iter)
    assert conv == bool(d["converged"])
    assert k == int(d["iterations"])
    ref = d["traj"]
    got = np.array(traj)
    assert got.shape == ref.shape
    assert np.array_equal(got[:, 0], ref[:, 0])
    assert rel_err(got[:, 1:], ref[:, 1:]) <= 1e-10
    assert rel_err(it.delta, d["delta"]) <= 1e-10


def test_bary_matches_reference():
    d = load("bary_grid5x5_m3")
    g = O.GridCost(5, 5, 2)
    prm = params_from(d["params"])
    margs = list(d["margs"])
    st = O.BaryIterate(d["in_deltas"].copy(), d["in_bs"].copy(), float(d["in_scalars"][0]),
                       float(d["in_scalars"][1]), int(d["in_scalars"][2]), d["w"], prm.eta)
    r = O.marginal_from_logz(st.w, O.log_normalizers(st.a, st.bs, g))
    assert rel_err(r, d["rmap"]) <= 1e-14
    nxt = O.bary_step(st, g, margs, prm)
    assert rel_err(nxt.deltas, d["out_deltas"]) <= 1e-13
    assert rel_err(nxt.bs, d["out_bs"]) <= 1e-13
    primal, dual, infeas, _ = O.bary_evaluate(st, g, margs)
    assert abs(primal - float(d["eval_primal"])) <= 1e-13
    assert abs(dual - float(d["eval_dual"])) <= 1e-13
    assert rel_err(infeas, d["eval_infeas"]) <= 1e-12
    st2, conv, k, traj, rbar = O.bary_solve(g, margs, d["w"], prm, eps=5e-3, max_iter=3000)
    assert conv == bool(d["solve_converged"]) and k == int(d["solve_iterations"])
    assert rel_err(rbar, d["solve_bary"]) <= 1e-10


def test_kat_spec_examples():
    d = load("kat_spec")
    assert np.allclose(d["implicit_row"], [0.75, 0.25], atol=1e-15)
    assert np.allclose(d["dual_md_step"], [0.8, -0.8], atol=1e-15)
    assert np.allclose(d["balance"], [np.log(3.0), np.log(1.5)], atol=1e-15)
    # oracle restatement reproduces the same examples
    prm = O.Params(0.0, 0.0, 1.0, 1.0, 1.1, 0.0)
    got = O._mirror(np.zeros(2), np.array([0.6, 0.4]), np.array([0.5, 0.5]), np.array([0.5, 0.5]), prm, 1.0)
    assert np.allclose(got, d["dual_md_step"], atol=0)


def test_hash_generator_properties():
    hc = O.HashCost(300, seed=7)
    blk = hc.block(0, 300)
    assert blk.shape == (300, 300)
    assert blk.max() == 1.0 and blk[0, 299] == 1.0
    assert 0.0 <= blk.min() < 0.01
    assert np.array_equal(hc.block(128, 200), blk[128:200])   # regenerable block by block
    assert not np.array_equal(O.HashCost(300, seed=8).block(1, 2), blk[1:2])


SINKHORN = golden_names("sinkhorn_")


@pytest.mark.parametrize("name", SINKHORN)
def test_sinkhorn_oracle_matches_reference(name):
    d = load(name)
    cost = oracle_cost(d)
    r, c = d["r"], d["c"]
    for eta, tol, mi in ((0.05, 1e-9, 10000), (0.01, 1e-8, 20000), (0.01, 1e-12, 7)):
        tag = f"eta{eta}_mi{mi}"
        phi, psi, conv, sweeps, gap = O.sinkhorn(cost, r, c, eta, tol=tol, max_iter=mi)
        info = d[f"{tag}_info"]
        assert conv == bool(info[0]) and sweeps == int(info[1])
        assert abs(gap - info[2]) <= 1e-12 + 1e-9 * info[2]
        assert rel_err(phi, d[f"{tag}_phi"]) <= 1e-12 and rel_err(psi, d[f"{tag}_psi"]) <= 1e-12
        assert abs(O.eot_dual(phi, psi, eta, cost, r, c) - float(d[f"{tag}_dual"])) <= 1e-12
        assert rel_err(O.sinkhorn_col(phi, psi, eta, cost), d[f"{tag}_col"]) <= 1e-12


def test_ibp_oracle_matches_reference():
    d = load("ibp_grid5x5_m3")
    g = O.GridCost(5, 5, 2)
    for eta, tol, mi in ((0.05, 1e-9, 5000), (0.02, 1e-12, 9)):
        tag = f"eta{eta}_mi{mi}"
        bary, phis, psis, conv, sweeps, gap, log_r = O.ibp(g, list(d["margs"]), d["w"], eta, tol=tol, max_iter=mi)
        info = d[f"{tag}_info"]
        assert conv == bool(info[0]) and sweeps == int(info[1])
        assert rel_err(bary, d[f"{tag}_bary"]) <= 1e-12
        assert rel_err(phis, d[f"{tag}_phis"]) <= 1e-12 and rel_err(psis, d[f"{tag}_psis"]) <= 1e-12


def test_oracle_pdxg_matches_reference_dense_iterate():
    """SPEC acceptance 1 needs the dense PDXG oracle (dxg.py:494-521): the oracle's restatement
    reproduces the reference's 500-iteration iterate (tests/golden/spec_acceptance.npz)."""
    d = load("spec_acceptance")
    for n in (4, 8, 16):
        p = d[f"pdxg{n}_params"]
        prm = O.Params(*[float(v) for v in p])
        C, r, c = d[f"pdxg{n}_C"], d[f"pdxg{n}_r"], d[f"pdxg{n}_c"]
        sup = 1.0
        Cn = C / C.max()
        delta, log_p = np.zeros(n), np.full((n, n), -np.log(n))
        for _ in range(500):
            delta, log_p = O.pdxg_step(delta, log_p, Cn, r, c, prm, sup)
        assert np.max(np.abs(log_p - d[f"pdxg{n}_log_p"])) <= 1e-11
        assert np.max(np.abs(delta - d[f"pdxg{n}_delta"])) <= 1e-11
