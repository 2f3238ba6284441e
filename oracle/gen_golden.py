"""Generate golden fixtures by running the REFERENCE (`leanot`) in the build container.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python oracle/gen_golden.py [--with-config1]

Writes tests/golden/*.npz.  The reference is not available on the GPU box, so its
outputs travel as these fixtures; tests compare both the oracle restatement
(CPU) and the CUDA path (GPU) against them.  Every fixture records the numpy
version and BLOCK_ROWS because the reference's summation order depends on them
(SURVEY.md §8c).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from leanot import barycenter as B  # noqa: E402
from leanot import core, dxg  # noqa: E402
from leanot import sinkhorn as SK  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def meta(**kw):
    return json.dumps({"numpy": np.__version__, "block_rows": core.BLOCK_ROWS, **kw})


def rand_hist(rng, n, zeros=0):
    w = rng.random(n) + 0.05
    if zeros:
        w[rng.choice(n, zeros, replace=False)] = 0.0
    return core.Histogram.normalized(w)


def kernels(rng):
    """Small instances for every CostKernel kind (core.py:200-288)."""
    out = {}
    out["explicit_n8"] = core.ExplicitKernel(rng.random((8, 8)))
    out["explicit_n37"] = core.ExplicitKernel(rng.random((37, 37)) * 3.0)
    out["explicit_n130"] = core.ExplicitKernel(rng.random((130, 130)))
    out["grid_6x5_p1"] = core.GridKernel(6, 5, 1)
    out["grid_7x9_p2"] = core.GridKernel(7, 9, 2)
    out["grid_4x4_p3"] = core.GridKernel(4, 4, 3)
    out["points_n50_d2_p2"] = core.ColorKernel(rng.random((50, 2)), 2)
    out["points_n45_d3_p2"] = core.ColorKernel(rng.random((45, 3)), 2)
    out["points_n33_d3_p1"] = core.ColorKernel(rng.random((33, 3)), 1)
    out["points_n20_d3_p3"] = core.ColorKernel(rng.random((20, 3)), 3)
    return out


def kernel_arrays(name, k):
    if isinstance(k, core.ExplicitKernel):
        return {"kind": "explicit", "C": k._m * k.scale}
    if isinstance(k, core.GridKernel):
        return {"kind": "grid", "H": k.height, "W": k.width, "p": k.p}
    return {"kind": "points", "F": k.features, "p": k.p}


def save(name, **arrays):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, len(arrays), "arrays")


def gen_sweeps(rng):
    """column_marginal / _plan_stats / dual / potentials on random states, every kernel kind."""
    ks = kernels(rng)
    for name, k in ks.items():
        n = k.n
        r = rand_hist(rng, n, zeros=1 if n > 30 else 0)
        c = rand_hist(rng, n)
        cases = []
        for trial in range(3):
            a = [0.0, 3.7, 250.0][trial]
            b = rng.normal(0, [0.0, 2.0, 40.0][trial], n)
            w = dxg.TransportLogWeights(a, b, 0.0, 0)
            delta = rng.uniform(-1.2, 1.2, n)
            mu = dxg.LogOddsField(delta)
            col = dxg.column_marginal(w, k, r)
            cost, col2, ent = dxg._plan_stats(w, k, r)
            prim0 = dxg.primal_penalized_value(w, k, r, c, 0.0)
            prim3 = dxg.primal_penalized_value(w, k, r, c, 1e-3)
            dual0 = dxg.dual_penalized_value(mu, k, r, c, 0.0)
            dual3 = dxg.dual_penalized_value(mu, k, r, c, 1e-3)
            dual7 = dxg.dual_penalized_value(mu, k, r, c, 1e-7)
            cases.append(dict(a=a, b=b, delta=delta, col=col, cost=cost, ent=ent, prim0=prim0,
                              prim3=prim3, dual0=dual0, dual3=dual3, dual7=dual7))
        rr = r if r.full_support else rand_hist(rng, n)
        pot = dxg.recover_eot_potentials(dxg.DxgState.initial(n), dxg.LogOddsField(cases[1]["delta"]),
                                         k, rr, 1e-2)
        arr = kernel_arrays(name, k)
        payload = {f"case{t}_{key}": np.asarray(v) for t, cs in enumerate(cases) for key, v in cs.items()}
        save(f"sweep_{name}", meta=meta(kind=arr.pop("kind"), scale=k.scale, sup_norm=k.sup_norm),
             r=r.weights, c=c.weights, r_full=rr.weights, pot_phi=pot.phi, pot_psi=pot.psi,
             **{f"k_{key}": np.asarray(v) for key, v in arr.items()}, **payload)


def gen_steps(rng):
    """dxg_step from injected states in every parameter regime (single-step parity)."""
    for name, k in (("explicit_n37", core.ExplicitKernel(rng.random((37, 37)))),
                    ("explicit_n200", core.ExplicitKernel(rng.random((200, 200)))),
                    ("grid_8x8_p1", core.GridKernel(8, 8, 1)),
                    ("points_n150_d2_p2", core.ColorKernel(rng.random((150, 2)), 2))):
        n = k.n
        r, c = rand_hist(rng, n), rand_hist(rng, n)
        schemes = {
            "tuned": dxg.params_tuned(0.0),
            "tuned_taumu005": dxg.params_tuned(0.0).with_overrides(tau_mu=0.05),
            "tuned_eta1e-3": dxg.params_tuned(1e-3),
            "loose": dxg.params_loose(n, 1e-2, c.min()),
            "li": dxg.params_li(n, 1e-2),
        }
        out = {"meta": meta(), "r": r.weights, "c": c.weights, **{f"k_{kk}": np.asarray(v) for kk, v in kernel_arrays(name, k).items() if kk != "kind"}}
        out["kind"] = np.asarray(kernel_arrays(name, k)["kind"])
        for sname, prm in schemes.items():
            state = dxg.DxgState(dxg.LogOddsField(rng.uniform(-1.1, 1.1, n)),
                                 dxg.TransportLogWeights(37.0, -np.abs(rng.normal(0, 30, n)), 0.25, 37))
            nxt = dxg.dxg_step(state, k, r, c, prm)
            out[f"{sname}_params"] = np.array([prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha])
            out[f"{sname}_in_delta"] = state.mu.delta
            out[f"{sname}_in_b"] = state.weights.b
            out[f"{sname}_in_scalars"] = np.array([state.weights.a, state.weights.s, state.weights.t])
            out[f"{sname}_out_delta"] = nxt.mu.delta
            out[f"{sname}_out_b"] = nxt.weights.b
            out[f"{sname}_out_scalars"] = np.array([nxt.weights.a, nxt.weights.s, nxt.weights.t])
            # a short trajectory from the zero state (per-iteration parity horizon)
            st = dxg.DxgState.initial(n)
            deltas, bs = [], []
            for _ in range(40):
                st = dxg.dxg_step(st, k, r, c, prm)
                deltas.append(st.mu.delta)
                bs.append(st.weights.b)
            out[f"{sname}_traj_delta"] = np.array(deltas)
            out[f"{sname}_traj_b"] = np.array(bs)
            out[f"{sname}_traj_scalars"] = np.array([st.weights.a, st.weights.s, st.weights.t])
        save(f"step_{name}", **out)


def gen_solves(rng):
    """Full solve trajectories in the non-chaotic regimes (same iteration count to eps)."""
    runs = []
    n = 64
    C = rng.random((n, n))
    r, c = rand_hist(rng, n), rand_hist(rng, n)
    runs.append(("explicit_n64_taumu005", core.ExplicitKernel(C), r, c,
                 dxg.params_tuned(0.0).with_overrides(tau_mu=0.05), dxg.Termination(eps=1e-4, max_iter=20000)))
    g = core.GridKernel(6, 6, 2)
    r2, c2 = rand_hist(rng, 36), rand_hist(rng, 36)
    runs.append(("grid_6x6_p2_loose", g, r2, c2, dxg.params_loose(36, 1e-2, c2.min()),
                 dxg.Termination(eps=1e-2, max_iter=20000)))
    f = rng.random((48, 2))
    r3, c3 = rand_hist(rng, 48), rand_hist(rng, 48)
    runs.append(("points_n48_eta1e-3_taumu005", core.ColorKernel(f, 2), r3, c3,
                 dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05), dxg.Termination(eps=1e-3, max_iter=20000)))
    runs.append(("explicit_n64_tuned_maxiter", core.ExplicitKernel(C), r, c, dxg.params_tuned(0.0),
                 dxg.Termination(eps=1e-10, max_iter=60)))
    for name, k, rr, cc, prm, term in runs:
        t0 = time.time()
        try:
            sol = dxg.solve(k, rr, cc, prm, term, log_stride=25, dense_cap=4096)
            rounding_failed = False
        except ValueError:  # Round can emit tiny negatives
            sol = dxg.solve(k, rr, cc, prm, term, log_stride=25, dense_cap=0)
            rounding_failed = True
        traj = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
        arr = kernel_arrays(name, k)
        save(f"solve_{name}", meta=meta(seconds=time.time() - t0, rounding_failed=rounding_failed), kind=np.asarray(arr.pop("kind")),
             **{f"k_{kk}": np.asarray(v) for kk, v in arr.items()},
             r=rr.weights, c=cc.weights,
             params=np.array([prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha]),
             term=np.array([term.eps, term.max_iter]), converged=np.asarray(sol.converged),
             iterations=np.asarray(sol.iterations), traj=traj, delta=sol.state.mu.delta,
             b=sol.state.weights.b, scalars=np.array([sol.state.weights.a, sol.state.weights.s, sol.state.weights.t]),
             col_gap=np.asarray(sol.report.col_gap),
             rounded_cost=np.asarray(np.nan if sol.rounded_cost is None else sol.rounded_cost),
             rounded_plan=(sol.rounded_plan.entries if sol.rounded_plan is not None else np.zeros((0, 0))))


def gen_config1():
    """BASELINE config 1: n=1000 random C, tuned + tau_mu=0.05, eps=1e-4 (8,225 iterations)."""
    n = 1000
    rng = np.random.default_rng(0)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    C = rng.random((n, n))
    k = core.ExplicitKernel(C)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    t0 = time.time()
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4), log_stride=25, workers=4, dense_cap=0)
    secs = time.time() - t0
    traj = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    save("config1_n1000", meta=meta(seconds=secs, workers=4), converged=np.asarray(sol.converged),
         iterations=np.asarray(sol.iterations), traj=traj, delta=sol.state.mu.delta, b=sol.state.weights.b,
         scalars=np.array([sol.state.weights.a, sol.state.weights.s, sol.state.weights.t]),
         col_gap=np.asarray(sol.report.col_gap))


def gen_bary(rng):
    """Barycenter: injected-state step, marginal map, objective, a short solve."""
    g = core.GridKernel(5, 5, 2)
    n, m = g.n, 3
    margs = [rand_hist(rng, n) for _ in range(m)]
    w = np.array([0.2, 0.5, 0.3])
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    st = B.BarycenterState.initial(n, w, prm.eta)
    st.deltas[:] = rng.uniform(-1, 1, (m, n))
    st.bs[:] = -np.abs(rng.normal(0, 5, (m, n)))
    st.a, st.s, st.t = 12.0, 0.11, 12
    nxt = B.dxgb_step(st, g, margs, prm)
    rmap = B.barycenter_marginal(st, g).weights
    obj = B.barycenter_objective(st, g, margs)
    primal, dual, infeas = B._bary_evaluate(st, g, margs, 1)
    sol = B.dxgb_solve(g, margs, w, prm, dxg.Termination(eps=5e-3, max_iter=3000), log_stride=25)
    traj = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    save("bary_grid5x5_m3", meta=meta(), margs=np.array([h.weights for h in margs]), w=w,
         params=np.array([prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha]),
         in_deltas=st.deltas, in_bs=st.bs, in_scalars=np.array([st.a, st.s, st.t]),
         out_deltas=nxt.deltas, out_bs=nxt.bs, out_scalars=np.array([nxt.a, nxt.s, nxt.t]),
         rmap=rmap, objective=np.asarray(obj), eval_primal=np.asarray(primal), eval_dual=np.asarray(dual),
         eval_infeas=infeas, solve_converged=np.asarray(sol.converged), solve_iterations=np.asarray(sol.iterations),
         solve_traj=traj, solve_bary=sol.barycenter.weights, solve_deltas=sol.state.deltas, solve_bs=sol.state.bs,
         solve_infeas=sol.per_marginal_infeas)


def gen_kat():
    """SPEC.md known-answer examples on the hot path."""
    kat = {}
    # implicit_row: a=0, b=(0, log 3) on n=2 -> (0.75, 0.25)
    kat["implicit_row"] = dxg.implicit_row(dxg.TransportLogWeights(0.0, np.array([0.0, np.log(3.0)]), 0.0, 0),
                                           core.ExplicitKernel(np.array([[0.0, 1.0], [1.0, 0.0]])), 0)
    # dual_md_step: delta=0, tau_mu=1, sup=1, c_tilde=0.5, residual 0.1 -> 0.8
    prm = dxg.DxgParams(eta=0.0, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.0)
    c = core.Histogram(np.array([0.5, 0.5]))
    kat["dual_md_step"] = dxg.dual_md_step(dxg.LogOddsField(np.zeros(2)), np.array([0.6, 0.4]), c,
                                           np.array([0.5, 0.5]), prm, 1.0).delta
    # balance: beta = log 3, delta = log 9 -> log 3
    kat["balance"] = dxg.balance(dxg.LogOddsField(np.array([np.log(9.0), np.log(1.5)])), np.log(3.0)).delta
    save("kat_spec", meta=meta(), **kat)


def gen_sinkhorn(rng):
    """Sinkhorn / IBP baselines (sinkhorn.py:74-228) -- SURVEY.md §8f item 1."""
    cases = {
        "explicit_n37": core.ExplicitKernel(rng.random((37, 37))),
        "grid_6x6_p2": core.GridKernel(6, 6, 2),
        "points_n40_d3_p2": core.ColorKernel(rng.random((40, 3)), 2),
    }
    for name, k in cases.items():
        n = k.n
        r, c = rand_hist(rng, n), rand_hist(rng, n)
        out = {"meta": meta(), "r": r.weights, "c": c.weights}
        arr = kernel_arrays(name, k)
        out["kind"] = np.asarray(arr.pop("kind"))
        out.update({f"k_{kk}": np.asarray(v) for kk, v in arr.items()})
        for eta, tol, mi in ((0.05, 1e-9, 10000), (0.01, 1e-8, 20000), (0.01, 1e-12, 7)):
            pot = SK.sinkhorn_solve(k, r, c, eta, tol=tol, max_iter=mi)
            tag = f"eta{eta}_mi{mi}"
            out[f"{tag}_phi"], out[f"{tag}_psi"] = pot.phi, pot.psi
            out[f"{tag}_info"] = np.array([pot.converged, pot.sweeps, pot.col_gap], dtype=float)
            out[f"{tag}_dual"] = np.asarray(SK.eot_dual_value(pot, k, r, c))
            out[f"{tag}_col"] = SK.sinkhorn_column_marginal(pot, k)
        save(f"sinkhorn_{name}", **out)
    g = core.GridKernel(5, 5, 2)
    margs = [rand_hist(rng, 25) for _ in range(3)]
    w = np.array([0.2, 0.5, 0.3])
    out = {"meta": meta(), "margs": np.array([h.weights for h in margs]), "w": w}
    for eta, tol, mi in ((0.05, 1e-9, 5000), (0.02, 1e-12, 9)):
        res = SK.ibp_barycenter(g, margs, w, eta, tol=tol, max_iter=mi)
        tag = f"eta{eta}_mi{mi}"
        out[f"{tag}_bary"] = res.barycenter.weights
        out[f"{tag}_phis"], out[f"{tag}_psis"] = res.phis, res.psis
        out[f"{tag}_info"] = np.array([res.converged, res.sweeps, res.col_gap], dtype=float)
        out[f"{tag}_logr"] = res.log_r
    save("ibp_grid5x5_m3", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-config1", action="store_true")
    args = ap.parse_args()
    rng = np.random.default_rng(20251114)
    gen_kat()
    gen_sweeps(rng)
    gen_steps(rng)
    gen_solves(rng)
    gen_bary(rng)
    gen_sinkhorn(np.random.default_rng(777))
    if args.with_config1:
        gen_config1()


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    main()
