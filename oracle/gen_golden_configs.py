"""Reference fixtures at BASELINE config shapes (runs the REFERENCE `leanot` in this container).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python oracle/gen_golden_configs.py {config2|hash4096|bary_grid} [--workers W]

config2    BASELINE config 2 at its full size: n = 1e4 2-D points, ColorKernel(f, p=2), the
           instance tools/bench_configs.py:config2 builds (seed 2), params_tuned(1e-6) +
           tau_mu = 0.05.  Runs dxg_step 50 times (dxg.py:261-279) and _evaluate at
           iterations 25 and 50 (dxg.py:412-417), i.e. exactly what solve(log_stride=25)
           does over its first 50 iterations, storing the iterates at 1, 2, 5, 10, 25, 50.
           (The full solve to eps = 1e-4 takes 31,675 iterations: ~17 h of reference CPU.)
hash4096   Iteration-count parity on the headline instance family: the bench's hash matrix
           (oracle.HashCost, BASELINE config 3's generator) at n = 4096, marginals as
           bench.py:marginals, tuned + tau_mu = 0.05, solve to eps = 1e-4 (dxg.py:420-472).
bary_grid  BASELINE config 5's instance family (tools/bench_configs.py:config5: Gaussian-
           mixture marginals, GridKernel(side, side, 2), m = 8, tuned(1e-3) + tau_mu = 0.05) at
           the largest sides the reference finishes in minutes: one dxgb_step, evaluation and
           r-map from an injected state at side 40 (n = 1600), dxgb_solve to eps = 1e-3 at side 16.

Writes tests/golden/<name>.npz.  Each records numpy's version and BLOCK_ROWS (the
reference's summation order depends on them).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from leanot import barycenter as B  # noqa: E402
from leanot import core, dxg  # noqa: E402

import leanot_oracle as O  # noqa: E402  (hash matrix generator only)

OUT = HERE.parent / "tests" / "golden"


def meta(**kw):
    return json.dumps({"numpy": np.__version__, "block_rows": core.BLOCK_ROWS, **kw})


def save(name, **arrays):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", OUT / f"{name}.npz", flush=True)


def hist(rng, n):
    w = rng.random(n)
    return w / w.sum()


def gen_config2(workers):
    n = 10_000
    rng = np.random.default_rng(2)
    f = rng.random((n, 2))
    k = core.ColorKernel(f, 2)
    r, c = core.Histogram(hist(rng, n)), core.Histogram(hist(rng, n))
    prm = dxg.params_tuned(1e-6).with_overrides(tau_mu=0.05)
    st = dxg.DxgState.initial(n)
    keep = {1, 2, 5, 10, 25, 50}
    out = {"features": f, "r": r.weights, "c": c.weights}
    evals = []
    t0 = time.time()
    for it in range(1, 51):
        st = dxg.dxg_step(st, k, r, c, prm, workers=workers)
        if it in keep:
            out[f"delta_{it}"] = st.mu.delta
            out[f"b_{it}"] = st.weights.b
            out[f"scal_{it}"] = np.array([st.weights.a, st.weights.s, float(st.weights.t)])
        if it % 25 == 0:
            p, d, inf = dxg._evaluate(st, k, r, c, prm.eta, workers)
            evals.append([it, p, d, p - d, inf, st.weights.s])
        print(f"config2 it {it} {time.time() - t0:.0f}s", flush=True)
    colm = dxg.column_marginal(st.weights, k, r, workers)
    save("config2_n1e4", meta=meta(seconds=time.time() - t0, workers=workers, seed=2, scale=k.scale),
         evals=np.array(evals), col_50=colm, **out)


def gen_hash4096(workers):
    n, seed = 4096, 0
    Cm = O.HashCost(n, seed).block(0, n)
    k = core.ExplicitKernel(Cm)
    rng = np.random.default_rng(seed + 1)   # bench.py:marginals
    rw, cw = rng.random(n), rng.random(n)
    r, c = core.Histogram(rw / rw.sum()), core.Histogram(cw / cw.sum())
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    t0 = time.time()
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4), log_stride=25, workers=workers, dense_cap=0)
    secs = time.time() - t0
    traj = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    save("hash4096_eps1e-4", meta=meta(seconds=secs, workers=workers, seed=seed), converged=np.asarray(sol.converged),
         iterations=np.asarray(sol.iterations), traj=traj, delta=sol.state.mu.delta, b=sol.state.weights.b,
         scalars=np.array([sol.state.weights.a, sol.state.weights.s, sol.state.weights.t]),
         col_gap=np.asarray(sol.report.col_gap))
    print("hash4096:", sol.iterations, sol.converged, f"{secs:.0f}s", flush=True)


def bary_instance(side, m=8, seed=5):
    """BASELINE config 5's instance builder (tools/bench_configs.py:config5) at grid side `side`:
    m Gaussian-mixture marginals (cli.py:401-408 _gaussian_mixture) + 1e-6, GridKernel(side, side, 2),
    uniform weights, params_tuned(1e-3) + tau_mu = 0.05."""
    rng = np.random.default_rng(seed)
    xs, ys = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    margs = []
    for _ in range(m):
        img = np.zeros((side, side))
        for _ in range(rng.integers(2, 5)):
            cx, cy = rng.uniform(0, side - 1, 2)
            sig = rng.uniform(side / 8.0, side / 3.0)
            img += rng.uniform(0.3, 1.0) * np.exp(-((xs - cx) ** 2 + (ys - cy) ** 2) / (2 * sig ** 2))
        h = img.ravel() / img.sum() + 1e-6
        margs.append(core.Histogram(h / h.sum()))
    k = core.GridKernel(side, side, 2)
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    return k, margs, np.full(m, 1.0 / m), prm


def gen_bary_grid(workers):
    """Step + evaluation from an injected state at side 40 (n = 1600, m = 8), solve at side 16."""
    m = 8
    out = {}
    k, margs, w, prm = bary_instance(40, m)
    n = k.n
    rng = np.random.default_rng(11)
    st = B.BarycenterState.initial(n, w, prm.eta)
    st.deltas[:] = rng.uniform(-0.5, 0.5, (m, n))
    st.bs[:] = -np.abs(rng.normal(0.0, 2.0, (m, n)))
    st.a, st.s, st.t = 7.0, 0.003, 7
    t0 = time.time()
    nxt = B.dxgb_step(st, k, margs, prm, workers=workers)
    primal, dual, infeas = B._bary_evaluate(nxt, k, margs, workers)
    rmap = B.barycenter_marginal(nxt, k, workers).weights
    out.update(margs40=np.array([h.weights for h in margs]), in_deltas=st.deltas, in_bs=st.bs,
               in_scalars=np.array([st.a, st.s, st.t]), out_deltas=nxt.deltas, out_bs=nxt.bs,
               out_scalars=np.array([nxt.a, nxt.s, nxt.t]), eval_primal=np.asarray(primal),
               eval_dual=np.asarray(dual), eval_infeas=infeas, rmap=rmap)
    k16, margs16, w16, prm16 = bary_instance(16, m)
    sol = B.dxgb_solve(k16, margs16, w16, prm16, dxg.Termination(eps=1e-3, max_iter=20000), log_stride=25,
                       workers=workers)
    traj = np.array([[p.iter, p.primal, p.dual, p.gap, p.col_infeas_l1, p.s] for p in sol.trajectory])
    secs = time.time() - t0
    save("bary_config5_shape", meta=meta(seconds=secs, workers=workers, m=m, sides=[40, 16]),
         params=np.array([prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha]),
         margs16=np.array([h.weights for h in margs16]), solve_converged=np.asarray(sol.converged),
         solve_iterations=np.asarray(sol.iterations), solve_traj=traj, solve_bary=sol.barycenter.weights,
         solve_infeas=sol.per_marginal_infeas, **out)
    print("bary_grid:", sol.iterations, sol.converged, f"{secs:.0f}s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["config2", "hash4096", "bary_grid"])
    ap.add_argument("--workers", type=int, default=4)
    a = ap.parse_args()
    {"config2": gen_config2, "hash4096": gen_hash4096, "bary_grid": gen_bary_grid}[a.which](a.workers)
