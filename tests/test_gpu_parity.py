"""CUDA path vs the reference's golden vectors and the oracle (needs a B200).

Tolerances (north_star): duals and marginals within 1e-10 relative per
iteration; final transport cost within 1e-8 relative; same iteration count to
eps.  Relative errors are norm-wise (max |x - ref| / max |ref|).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import device_cost, golden_names, load, oracle_cost, params_from, rel_err

pytestmark = pytest.mark.gpu

SWEEPS = golden_names("sweep_")
STEPS = golden_names("step_")
SOLVES = golden_names("solve_")
TOL_ITER = 1e-10


def _dxg():
    from paper_2511_11359_b200 import dxg
    return dxg


@pytest.mark.parametrize("name", SWEEPS)
def test_column_marginal_vs_reference(name):
    dxg = _dxg()
    d = load(name)
    k = device_cost(d)
    for t in range(3):
        w = dxg.TransportLogWeights(float(d[f"case{t}_a"]), d[f"case{t}_b"], 0.0, 0)
        col = dxg.column_marginal(w, k, d["r"])
        assert rel_err(col, d[f"case{t}_col"]) <= 1e-13, t
        assert abs(col.sum() - 1.0) <= 1e-12


@pytest.mark.parametrize("name", SWEEPS)
def test_evaluation_functions_vs_reference(name):
    dxg = _dxg()
    d = load(name)
    k = device_cost(d)
    r, c = d["r"], d["c"]
    for t in range(3):
        w = dxg.TransportLogWeights(float(d[f"case{t}_a"]), d[f"case{t}_b"], 0.0, 0)
        mu = dxg.LogOddsField(d[f"case{t}_delta"])
        cost, col, ent = dxg._plan_stats(w, k, r)
        assert abs(cost - float(d[f"case{t}_cost"])) <= 1e-13 * max(1, abs(cost))
        assert abs(ent - float(d[f"case{t}_ent"])) <= 1e-12 * max(1, abs(ent))
        assert abs(dxg.primal_penalized_value(w, k, r, c, 0.0) - float(d[f"case{t}_prim0"])) <= 1e-12
        assert abs(dxg.primal_penalized_value(w, k, r, c, 1e-3) - float(d[f"case{t}_prim3"])) <= 1e-12
        assert abs(dxg.dual_penalized_value(mu, k, r, c, 0.0) - float(d[f"case{t}_dual0"])) <= 1e-13
        assert abs(dxg.dual_penalized_value(mu, k, r, c, 1e-3) - float(d[f"case{t}_dual3"])) <= 1e-12
        assert abs(dxg.dual_penalized_value(mu, k, r, c, 1e-7) - float(d[f"case{t}_dual7"])) <= 1e-12
    pot = dxg.recover_eot_potentials(dxg.DxgState.initial(k.n), dxg.LogOddsField(d["case1_delta"]), k,
                                     d["r_full"], 1e-2)
    assert rel_err(pot.phi, d["pot_phi"]) <= 1e-11
    assert rel_err(pot.psi, d["pot_psi"]) <= 1e-14


SCHEMES = ["tuned", "tuned_taumu005", "tuned_eta1e-3", "loose", "li"]


@pytest.mark.parametrize("name", STEPS)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_dxg_step_injected_state(name, scheme):
    """Single-step parity from injected states: valid in every regime, chaotic ones included."""
    dxg = _dxg()
    d = load(name)
    k = device_cost(d)
    prm = dxg.DxgParams(*[float(v) for v in d[f"{scheme}_params"]])
    a, s, t = d[f"{scheme}_in_scalars"]
    st = dxg.DxgState(dxg.LogOddsField(d[f"{scheme}_in_delta"]),
                      dxg.TransportLogWeights(float(a), d[f"{scheme}_in_b"], float(s), int(t)))
    nxt = dxg.dxg_step(st, k, d["r"], d["c"], prm)
    assert rel_err(nxt.mu.delta, d[f"{scheme}_out_delta"]) <= TOL_ITER
    assert rel_err(nxt.weights.b, d[f"{scheme}_out_b"]) <= TOL_ITER
    assert [nxt.weights.a, nxt.weights.s, nxt.weights.t] == d[f"{scheme}_out_scalars"].tolist()


# Per-iteration horizons: params_li (tau_mu ~ 450) amplifies rounding noise the way
# tuned tau_mu=1 does -- the reference itself, with only its row-block size changed,
# leaves 1e-10 after ~20 iterations (tests/test_oracle_noise.py) -- so li is compared
# over its first 12 iterations; the other regimes over all 40.
HORIZON = {"tuned_taumu005": 40, "loose": 40, "tuned_eta1e-3": 40, "li": 12}


@pytest.mark.parametrize("name", STEPS)
@pytest.mark.parametrize("scheme", ["tuned_taumu005", "loose", "li", "tuned_eta1e-3"])
def test_trajectory_per_iteration(name, scheme):
    """Iterations from the zero state through the solver engine, every iterate within 1e-10."""
    from paper_2511_11359_b200.engine import DxgEngine
    d = load(name)
    k = device_cost(d)
    dxg = _dxg()
    prm = dxg.DxgParams(*[float(v) for v in d[f"{scheme}_params"]])
    eng = DxgEngine(k, d["r"], d["c"], prm)
    n = k.n
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    steps = d[f"{scheme}_traj_delta"].shape[0]
    for it in range(steps):
        eng.sweep()
        eng.update()
        delta, b, a, s, t = eng.read_state()
        if it < HORIZON[scheme]:
            assert rel_err(delta, d[f"{scheme}_traj_delta"][it]) <= TOL_ITER, it
            assert rel_err(b, d[f"{scheme}_traj_b"][it]) <= TOL_ITER, it
    assert [a, s, t] == d[f"{scheme}_traj_scalars"].tolist()


@pytest.mark.parametrize("name", SOLVES + [s + "@graph" for s in SOLVES if "points" in s])
def test_solve_vs_reference(name, monkeypatch):
    """Same iteration count, same converged flag, trajectory and final cost.  "@graph": the
    launch-per-kernel path (CUDA graph of sweeps + updates) instead of the persistent small-n
    kernel, i.e. the expanded-form sweeps for squared-Euclidean points."""
    if name.endswith("@graph"):
        name = name[: -len("@graph")]
        monkeypatch.setenv("LEANOT_PERSIST", "0")
    dxg = _dxg()
    d = load(name)
    k = device_cost(d)
    prm = dxg.DxgParams(*[float(v) for v in d["params"]])
    term = dxg.Termination(eps=float(d["term"][0]), max_iter=int(d["term"][1]))
    sol = dxg.solve(k, d["r"], d["c"], prm, term, log_stride=25, dense_cap=0)
    assert sol.iterations == int(d["iterations"])
    assert sol.converged == bool(d["converged"])
    got = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    ref = d["traj"]
    assert got.shape == ref.shape and np.array_equal(got[:, 0], ref[:, 0])
    if "tuned_maxiter" not in name:
        assert rel_err(got[:, 1], ref[:, 1]) <= 1e-8       # primal (transport cost)
        assert rel_err(got[:, 2], ref[:, 2]) <= 1e-8
        assert rel_err(sol.state.mu.delta, d["delta"]) <= 1e-8
    assert abs(sol.report.col_gap - float(d["col_gap"])) <= 1e-8 * max(1.0, float(d["col_gap"])) + 1e-14


def test_hash_kernel_matches_oracle_bits():
    from paper_2511_11359_b200 import core
    hk = core.HashKernel(1001, seed=3)
    hc = O.HashCost(1001, seed=3)
    for i0, i1 in ((0, 5), (500, 503), (998, 1001)):
        assert np.array_equal(hk.block(i0, i1), hc.block(i0, i1))


@pytest.mark.parametrize("n", [1, 2, 3, 17, 513, 1000])
def test_random_sizes_vs_oracle(n):
    """Ragged sizes (odd n, partial tiles) against the oracle."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    rng = np.random.default_rng(n)
    Cm = rng.random((n, n)) * 5
    r = O.normalized_hist(rng.random(n))
    c = O.normalized_hist(rng.random(n))
    k = core.ExplicitKernel(Cm)
    ok = O.DenseCost(Cm)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    st = dxg.DxgState(dxg.LogOddsField(rng.uniform(-1, 1, n)),
                      dxg.TransportLogWeights(40.0, -np.abs(rng.normal(0, 20, n)), 0.0, 40))
    nxt = dxg.dxg_step(st, k, r, c, prm)
    onxt = O.step(O.Iterate(st.mu.delta, 40.0, st.weights.b, 0.0, 40), ok, r, c,
                  O.params_tuned(0.0, tau_mu=0.05))
    assert rel_err(nxt.mu.delta, onxt.delta) <= TOL_ITER
    assert rel_err(nxt.weights.b, onxt.b) <= TOL_ITER


def test_zero_cost_and_sparse_marginal():
    """C == 0 (sup_norm 0) and r with zeros: the SPEC fixed point."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    n = 40
    k = core.ExplicitKernel(np.zeros((n, n)))
    assert k.sup_norm == 0.0 and k.scale == 1.0
    r = np.zeros(n)
    r[:10] = 0.1
    c = np.full(n, 1.0 / n)
    prm = dxg.params_tuned(0.0)
    st = dxg.DxgState.initial(n)
    for _ in range(3):
        st = dxg.dxg_step(st, k, r, c, prm)
    assert np.allclose(st.mu.delta, 0.0, atol=1e-14)
    col = dxg.column_marginal(st.weights, k, r)
    assert np.allclose(col, 1.0 / n, atol=1e-15)


def test_large_dynamic_range_shift_fixup():
    """Injected state far from any previous shift: rows must be recomputed exactly."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    n = 300
    rng = np.random.default_rng(5)
    Cm = rng.random((n, n))
    k = core.ExplicitKernel(Cm)
    r = O.normalized_hist(rng.random(n))
    for a, bscale in ((3000.0, 1500.0), (1e5, 10.0), (0.0, 900.0)):
        b = -np.abs(rng.normal(0, bscale, n))
        col = dxg.column_marginal(dxg.TransportLogWeights(a, b, 0.0, 0), k, r)
        (ref,) = O.column_marginals(O.DenseCost(Cm), r, [(a, b)])
        assert rel_err(col, ref) <= 1e-11


def test_config1_same_iteration_count_as_reference():
    """BASELINE config 1 end to end: n=1000 random C, tuned + tau_mu=0.05, eps=1e-4.

    The reference converges at iteration 8,225 (tests/golden/config1_n1000.npz)."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    d = load("config1_n1000")
    n = 1000
    rng = np.random.default_rng(0)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    Cm = rng.random((n, n))
    k = core.ExplicitKernel(Cm)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4), log_stride=25, dense_cap=0)
    assert sol.converged and sol.iterations == int(d["iterations"]) == 8225
    ref = d["traj"]
    got = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    assert got.shape == ref.shape
    assert rel_err(got[:, 1], ref[:, 1]) <= 1e-8
    assert rel_err(got[:, 2], ref[:, 2]) <= 1e-8
    assert abs(sol.final.primal - ref[-1, 1]) <= 1e-8 * abs(ref[-1, 1])   # final transport cost
    assert rel_err(sol.state.mu.delta, d["delta"]) <= 1e-8


@pytest.mark.parametrize("kind,n", [("explicit", 1000), ("points", 513), ("explicit", 37)])
def test_persistent_iterations_match_launch_per_kernel_path(kind, n):
    """n <= 4096: leanot_dxg_iterate runs all iterations in one cooperative kernel; it must
    track the regular kernels (graph of sweep + update launches) iteration by iteration."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200.engine import DxgEngine
    rng = np.random.default_rng(n)
    k = core.ExplicitKernel(rng.random((n, n))) if kind == "explicit" else core.ColorKernel(rng.random((n, 3)), 2)
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 30, n))
    b -= b.max()
    out = []
    for graph in (False, True):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(delta, b, 60.0, 0.1, 60)
        eng.iterate(50, use_graph=graph)
        out.append(eng.read_state())
    (d0, b0, a0, s0, t0), (d1, b1, a1, s1, t1) = out
    assert rel_err(d0, d1) <= 1e-11 and rel_err(b0, b1) <= 1e-11
    assert a0 == a1 and s0 == s1 and t0 == t1 == 110


@pytest.mark.parametrize("n", [500, 2000])
def test_persistent_paths_recompute_out_of_range_rows(n):
    """A jump in a after the shifts were set (every row sum far outside [2^-900, 2^900]) forces
    the exact-max recompute inside the persistent kernels (row-owner for n <= 1024, the
    four-barrier one above): they must track the launch-per-kernel path."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    from paper_2511_11359_b200.engine import DxgEngine
    rng = np.random.default_rng(n + 7)
    k = core.ExplicitKernel(rng.random((n, n)))
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 5, n))
    b -= b.max()
    out = []
    for graph in (False, True):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(delta, b, 10.0, 0.0, 10)
        eng.scal[0] = 1.0e6                  # x - m ~ -1e6 min_j C_ij: row sums underflow
        eng.scal[1] = 1.0e6 + prm.tau_p
        eng.iterate(6, use_graph=graph)
        out.append(eng.read_state())
    (d0, b0, a0, s0, t0), (d1, b1, a1, s1, t1) = out
    assert np.all(np.isfinite(d0)) and np.all(np.isfinite(b0))
    assert rel_err(d0, d1) <= 1e-11 and rel_err(b0, b1) <= 1e-11
    assert a0 == a1 and t0 == t1 == 16


@pytest.mark.parametrize("n,p", [(1200, 2), (1201, 1), (2500, 2)])
def test_pass_a_wave_tail_split_vs_oracle(n, p):
    """Point costs at sizes whose last pass-A wave is split into half-height row blocks
    (launch_rowpass_t: n = 1200 -> 296 four-row blocks + 2 two-row blocks); the step must
    match the oracle exactly as for unsplit sizes."""
    dxg = _dxg()
    from paper_2511_11359_b200 import core
    rng = np.random.default_rng(n)
    f = rng.random((n, 2))
    r = O.normalized_hist(rng.random(n))
    c = O.normalized_hist(rng.random(n))
    k = core.ColorKernel(f, p)
    ok = O.PointCost(f, p)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    st = dxg.DxgState(dxg.LogOddsField(rng.uniform(-1, 1, n)),
                      dxg.TransportLogWeights(40.0, -np.abs(rng.normal(0, 20, n)), 0.0, 40))
    nxt = dxg.dxg_step(st, k, r, c, prm)
    onxt = O.step(O.Iterate(st.mu.delta, 40.0, st.weights.b, 0.0, 40), ok, r, c,
                  O.params_tuned(0.0, tau_mu=0.05))
    assert rel_err(nxt.mu.delta, onxt.delta) <= TOL_ITER
    assert rel_err(nxt.weights.b, onxt.b) <= TOL_ITER
