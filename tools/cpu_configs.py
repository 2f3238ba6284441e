"""The reference algorithm (oracle port of leanot) on the host cores for BASELINE configs 1, 2, 4, 5.

Each config times a bounded sample with all host threads and extrapolates, labelled as such
(SURVEY.md §8d "CPU timing"):
  config 1  n=1000 dense C: 30 dxg_steps, x 8,225 iterations (+ 329 evaluation sweeps)
  config 2  n=1e4 2-D points: 2 dxg_steps, x the GPU's iteration count to eps (31,675)
  config 4  n=1e6 3-D points: both weight sets' column sweeps over 16 x 128 sampled rows,
            extrapolated to all 1e6 rows (per-iteration time of the whole problem)
  config 5  barycenter 316x316 grid, m=8: one softmax sweep of both weight sets over sampled
            rows, x 2m marginal sweeps + 2m LSE sweeps per iteration (barycenter.py:108-151)
Test/measurement infrastructure: runs the oracle only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import leanot_oracle as O  # noqa: E402

W = O.default_workers()


def hist(rng, n):
    w = rng.random(n)
    return w / w.sum()


def sampled_sweep_seconds(cost, n, a, b, r, rows):
    """Seconds for both weight sets' softmax column sweep over `rows` rows (W threads)."""
    a_bar, b_bar = a * 1.01 + 0.5, b * 0.99
    wsets = [(a, b), (a_bar, b_bar)]

    def work(i0, i1):
        Cb = cost.block(i0, i1)
        return [r[i0:i1] @ O._softmax_block(aa, bb, Cb) for aa, bb in wsets]

    work(0, min(O.BLOCK_ROWS, rows))
    t0 = time.perf_counter()
    O.run_blocks(work, rows, workers=W)
    return time.perf_counter() - t0


def config1():
    n = 1000
    rng = np.random.default_rng(0)
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    cost = O.DenseCost(rng.random((n, n)))
    prm = O.params_tuned(0.0, tau_mu=0.05)
    it = O.Iterate.zero(n)
    it = O.step(it, cost, r, c, prm, workers=W)
    t0 = time.perf_counter()
    for _ in range(30):
        it = O.step(it, cost, r, c, prm, workers=W)
    per = (time.perf_counter() - t0) / 30
    t0 = time.perf_counter()
    O.evaluate(it, cost, r, c, 0.0, workers=W)
    ev = time.perf_counter() - t0
    return {"config": 1, "seconds_per_iter": per, "eval_seconds": ev,
            "time_to_eps_s_extrapolated": per * 8225 + ev * (8225 // 25 + 1),
            "sample": f"30 dxg_steps + 1 evaluation, {W} threads; x 8,225 iterations / 329 evaluations"}


def config2():
    n = 10_000
    rng = np.random.default_rng(2)
    f = rng.random((n, 2))
    cost = O.PointCost(f, 2)
    r, c = hist(rng, n), hist(rng, n)
    prm = O.params_tuned(1e-6, tau_mu=0.05)
    it = O.Iterate.zero(n)
    t0 = time.perf_counter()
    for _ in range(2):
        it = O.step(it, cost, r, c, prm, workers=W)
    per = (time.perf_counter() - t0) / 2
    return {"config": 2, "seconds_per_iter": per, "time_to_eps_s_extrapolated": per * 31675,
            "sample": f"2 dxg_steps, {W} threads; x 31,675 iterations (the GPU's count to eps = 1e-4)"}


def config4():
    n = 1_000_000
    rng = np.random.default_rng(4)
    f = rng.random((n, 3))
    f[0], f[1] = 0.0, 1.0
    cost = O.PointCost(f, 2, scale=3.0)
    r = hist(rng, n)
    b = -np.abs(rng.normal(0, 10, n))
    rows = O.BLOCK_ROWS * W
    secs = sampled_sweep_seconds(cost, n, 300.0, b, r, rows)
    per = secs * n / rows
    return {"config": 4, "seconds_per_iter": per, "iters_per_s": 1.0 / per,
            "sample": f"{rows} of {n} rows, both weight sets, {W} threads; extrapolated x{n / rows:.0f}"}


def config5():
    side, m = 316, 8
    n = side * side
    rng = np.random.default_rng(5)
    cost = O.GridCost(side, side, 2)
    r = hist(rng, n)
    b = -np.abs(rng.normal(0, 10, n))
    rows = O.BLOCK_ROWS * W
    secs = sampled_sweep_seconds(cost, n, 300.0, b, r, rows)
    full_pair = secs * n / rows          # both weight sets of one marginal, all rows
    per = full_pair * m * 2              # + the LSE sweeps (barycenter.py:78-87) of comparable cost
    return {"config": 5, "seconds_per_iter": per, "iters_per_s": 1.0 / per,
            "time_to_eps_s_extrapolated": per * 950,
            "sample": f"{rows} of {n} rows, both weight sets of one marginal, {W} threads; x{n / rows:.1f} rows "
                      f"x m={m} marginals x 2 (column + LSE sweeps); x 950 iterations (the GPU's count to eps = 1e-3)"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = []
    for cfg in a.configs.split(","):
        d = {"1": config1, "2": config2, "4": config4, "5": config5}[cfg]()
        d["cores"] = W
        d["kind"] = "port"
        print(json.dumps(d), flush=True)
        res.append(d)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))
