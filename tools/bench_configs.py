"""Per-configuration measurements for BASELINE.json configs 1, 2, 4 (per-GPU shard), 5 on one B200.

Writes one JSON object per config to stdout (and --out).  bench.py stays the single
headline line (config 3); this script backs DESIGN.md / profiles/ with the rest.

  config 1  n=1000 random C, tuned+tau_mu=0.05, eps=1e-4: time-to-eps, iterations (reference: 8,225)
  config 2  n=1e4 2-D points (on the fly), tuned(1e-6)+tau_mu=0.05, eps=1e-4: iters/s + time-to-eps
  config 4  n=1e6 3-D points (on the fly): one 1/8 row shard (the per-GPU work of the 8-GPU run)
  config 5  barycenter, GridKernel(316,316,2), m=8 Gaussian-mixture marginals, eta=1e-3: iters/s
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import torch  # noqa: E402

from paper_2511_11359_b200 import barycenter as B  # noqa: E402
from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine, shard_rows  # noqa: E402


def timed_iters(eng, iters):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        eng.sweep()
        eng.update()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / iters


def hist(rng, n):
    w = rng.random(n)
    return w / w.sum()


def config1():
    n = 1000
    rng = np.random.default_rng(0)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    k = core.ExplicitKernel(rng.random((n, n)))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4, max_iter=50), dense_cap=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4), dense_cap=0)
    secs = time.perf_counter() - t0
    return {"config": 1, "n": n, "time_to_eps_s": secs, "iterations": sol.iterations, "converged": sol.converged,
            "reference_iterations": 8225, "iters_per_s": sol.iterations / secs, "final_primal": sol.final.primal}


def config2(timeout):
    n = 10_000
    rng = np.random.default_rng(2)
    f = rng.random((n, 2))
    k = core.ColorKernel(f, 2)
    r, c = core.Histogram(hist(rng, n)), core.Histogram(hist(rng, n))
    prm = dxg.params_tuned(1e-6).with_overrides(tau_mu=0.05)
    eng = DxgEngine(k, r.weights, c.weights, prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    timed_iters(eng, 10)             # warm-up (lazy kernel attributes, occupancy queries)
    per_iter = timed_iters(eng, 200)
    t0 = time.perf_counter()
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4, timeout=None, max_iter=int(timeout / per_iter)),
                    dense_cap=0)
    secs = time.perf_counter() - t0
    return {"config": 2, "n": n, "cost": "2-D points p=2 on the fly", "iters_per_s": 1.0 / per_iter,
            "solve_seconds": secs, "iterations": sol.iterations, "converged": sol.converged,
            "final_gap": sol.final.gap, "final_infeas": sol.final.col_infeas_l1}


def config4(shards=8):
    n = 1_000_000
    rng = np.random.default_rng(4)
    f = rng.random((n, 3))
    f[0] = 0.0
    f[1] = 1.0                       # cube corners: raw sup = 3 by construction
    k = core.ColorKernel(f, 2, scale=3.0)
    r0, r1 = shard_rows(n, shards, 0)
    k.row0, k.row1 = r0, r1          # this GPU's rows (the per-GPU work of the sharded run)
    prm = dxg.params_tuned(1e-7).with_overrides(tau_mu=0.05)
    eng = DxgEngine(k, hist(rng, n), hist(rng, n), prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    eng.sweep(); eng.update()
    per_iter = timed_iters(eng, 2)
    # FP64 instructions per element and pass (expanded form, csrc/leanot_cost.cuh CostGram<3>):
    # dot product 3 (DMUL + 2 DFMA) + per weight set: x' 1 + table exp 7 (incl. the accumulate)
    per_elem = 2 * (3 + 2 * 8)
    fp64 = per_elem * n * (r1 - r0) / per_iter
    # SURVEY.md §8(d) algorithmic count for config 4: 47 FP64 instructions per element and
    # iteration (single-read ideal with libdevice exps); reported beside the executed count
    alg = 47 * n * (r1 - r0) / per_iter
    return {"config": 4, "n": n, "rows_this_gpu": r1 - r0, "shards": shards, "seconds_per_iter_per_gpu": per_iter,
            "projected_iters_per_s_8gpu": 1.0 / per_iter, "fp64_instr_per_s": fp64,
            "fp64_instr_per_element_iter": per_elem, "fp64_frac_of_measured_dfma_peak": fp64 / 17.07e12,
            "fp64_frac_survey_count": alg / 17.07e12,
            "fp64_definitions": "executed: 38 FP64 instructions per element and iteration in the two-pass "
                                "expanded form (what the kernels issue); survey: SURVEY.md §8(d)'s 47 per element "
                                "(single-read, libdevice exp); peak: builder DFMA microbenchmark 17.07e12/s at "
                                "1965 MHz (profiles/r01_microbench.md), not in MEASURED_PEAKS.json",
            "note": "1 GPU runs one 1/8 row shard; the 8-GPU run adds one 16 MB all-gather per iteration"}


def config5(tte5=0.0):
    sys.path.insert(0, str(ROOT / "oracle"))
    side, m = 316, 8
    n = side * side
    rng = np.random.default_rng(5)
    xs, ys = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    margs = []
    for _ in range(m):   # cli._gaussian_mixture (cli.py:401-408) + 1e-6 perturbation (core.py:147-164)
        img = np.zeros((side, side))
        for _ in range(rng.integers(2, 5)):
            cx, cy = rng.uniform(0, side - 1, 2)
            sig = rng.uniform(side / 8.0, side / 3.0)
            img += rng.uniform(0.3, 1.0) * np.exp(-((xs - cx) ** 2 + (ys - cy) ** 2) / (2 * sig ** 2))
        h = img.ravel() / img.sum() + 1e-6
        margs.append(core.Histogram(h / h.sum()))
    g = core.GridKernel(side, side, 2)
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    eng = B.BaryEngine(g, margs, np.full(m, 1.0 / m), prm)
    eng.load_state(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, fresh=True)
    eng.sweep(); eng.update()
    per_iter = timed_iters(eng, 5)
    out = {"config": 5, "n": n, "m": m, "cost": "GridKernel(316,316,2): separable O(n^1.5) sweeps",
           "seconds_per_iter": per_iter, "iters_per_s": 1.0 / per_iter}
    if tte5 > 0:
        # the IBP baseline (sinkhorn.py:174-228) on the same instance, separable sweeps
        from paper_2511_11359_b200 import sinkhorn as SK
        SK.ibp_barycenter(g, margs, np.full(m, 1.0 / m), 1e-3, tol=1e-9, max_iter=3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ib = SK.ibp_barycenter(g, margs, np.full(m, 1.0 / m), 1e-3, tol=1e-9, max_iter=2000)
        out.update({"ibp_eta": 1e-3, "ibp_seconds": time.perf_counter() - t0, "ibp_sweeps": ib.sweeps,
                    "ibp_converged": ib.converged, "ibp_col_gap": ib.col_gap})
        t0 = time.perf_counter()
        sol = B.dxgb_solve(g, margs, np.full(m, 1.0 / m), prm,   # no timeout: no per-iteration host sync
                           dxg.Termination(eps=1e-3, max_iter=int(tte5 / per_iter)), log_stride=25)
        out.update({"eps": 1e-3, "solve_seconds": time.perf_counter() - t0, "iterations": sol.iterations,
                    "converged": sol.converged, "final_gap": sol.final.gap, "final_max_infeas": sol.final.col_infeas_l1})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--timeout2", type=float, default=60.0)
    ap.add_argument("--tte5", type=float, default=300.0, help="config-5 solve wall-time budget (s), 0 = skip")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = []
    for cfg in a.configs.split(","):
        fn = {"1": config1, "2": lambda: config2(a.timeout2), "4": config4, "5": lambda: config5(a.tte5)}[cfg]
        t0 = time.perf_counter()
        d = fn()
        d["wall_s"] = time.perf_counter() - t0
        print(json.dumps(d), flush=True)
        res.append(d)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))
