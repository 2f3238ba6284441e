"""Small-n runs of every kernel family for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_small.py --case tma

Cases (each a few sweeps at small n so the instrumented run stays short):
  tma        stored cost, even n: rowpass_tma_kernel (cp.async.bulk + mbarrier ring) + colpass +
             slab reduce + O(n) updates + an evaluation sweep with forced fixup rows
  points     on-the-fly point costs: expanded-form (Gram) and difference-form sweeps
  rowowner   n <= 1024: the persistent row-owner kernel (cooperative, 2 grid barriers / iteration)
  persist    1024 < n <= 4096: the persistent iterate kernel (cooperative grid barriers)
  fused      stored cost, n = 16384: the L2-reuse single-launch sweep (release/acquire counters)
  sr         the single-read sweep forced at n = 2048 (tagged global exchange, mbarriers)
  sep        separable grid path (DMMA GEMM, cp.async ring) for DXG and the barycenter
  bary       dense barycenter sweeps + r-map
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import torch  # noqa: E402

from paper_2511_11359_b200 import barycenter as B  # noqa: E402
from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402


def hist(rng, n):
    w = rng.random(n) + 0.05
    return w / w.sum()


def state(rng, n, a=30.0):
    b = -np.abs(rng.normal(0, 2.0, n))
    return rng.uniform(-1, 1, n), b - b.max(), a, 0.1, 30


def engine_run(k, n, rng, eta=0.0, fused=False, single_read=None, iters=3):
    prm = dxg.params_tuned(eta).with_overrides(tau_mu=0.05)
    eng = DxgEngine(k, hist(rng, n), hist(rng, n), prm)
    eng.load_state(*state(rng, n))
    for _ in range(iters):
        eng.sweep(fused=fused, single_read=single_read)
        eng.update()
    eng.scal[0] = 2000.0           # force fixup rows on the evaluation sweep
    eng.sweep(evaluate=True)
    eng.evaluate()
    torch.cuda.synchronize()


def main(case):
    rng = np.random.default_rng(0)
    if case == "tma":
        engine_run(core.HashKernel(2048, seed=1), 2048, rng)
    elif case == "points":
        f = rng.random((3000, 3))
        engine_run(core.ColorKernel(f, 2), 3000, rng, eta=1e-3)
        k = core.ColorKernel(f, 2)
        k.norms_dev = None
        engine_run(k, 3000, rng)
    elif case == "rowowner":
        n = 600
        k = core.ExplicitKernel(rng.random((n, n)))
        sol = dxg.solve(k, core.Histogram(hist(rng, n)), core.Histogram(hist(rng, n)),
                        dxg.params_tuned(0.0).with_overrides(tau_mu=0.05), dxg.Termination(eps=1e-12, max_iter=50),
                        dense_cap=0)
        assert sol.iterations == 50
    elif case == "persist":
        n = 2500
        k = core.HashKernel(n, seed=2)
        prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
        eng = DxgEngine(k, hist(rng, n), hist(rng, n), prm)
        eng.load_state(*state(rng, n))
        eng.sweep()
        eng.update()
        eng.iterate(10, use_graph=False)
        torch.cuda.synchronize()
    elif case == "fused":
        engine_run(core.HashKernel(16384, seed=3), 16384, rng, fused=True, iters=1)
    elif case == "sr":
        engine_run(core.HashKernel(2048, seed=4), 2048, rng, single_read=True)
    elif case == "sep":
        g = core.GridKernel(16, 16, 2)
        engine_run(g, g.n, rng, eta=1e-3)
        margs = [core.Histogram(hist(rng, g.n)) for _ in range(3)]
        B.dxgb_solve(g, margs, np.array([0.2, 0.5, 0.3]), dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05),
                     dxg.Termination(eps=1e-12, max_iter=30), log_stride=10)
    elif case == "bary":
        k = core.ColorKernel(rng.random((700, 2)), 2)
        margs = [core.Histogram(hist(rng, 700)) for _ in range(3)]
        B.dxgb_solve(k, margs, np.array([0.2, 0.5, 0.3]), dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05),
                     dxg.Termination(eps=1e-12, max_iter=30), log_stride=10)
    torch.cuda.synchronize()
    print("case", case, "ok", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    main(ap.parse_args().case)
