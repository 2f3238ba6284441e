"""A/B: dense barycenter iterations with two marginals per read of C vs one (LEANOT_BARY_BATCH).

    python tools/bary_ab.py

Stored cost (n = 20,000, 3.2 GB in HBM) and 2-D point cloud (n = 10,000, on the fly), m = 8
marginals, tuned(1e-2) + tau_mu = 0.05, CUDA events around 10 plain iterations (sweep + update).
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import torch  # noqa: E402

from paper_2511_11359_b200 import barycenter as B  # noqa: E402
from paper_2511_11359_b200 import core, dxg  # noqa: E402


def run(kind, batch, m=8, iters=10):
    os.environ["LEANOT_BARY_BATCH"] = batch
    rng = np.random.default_rng(7)
    if kind == "stored":
        n = 20000
        k = core.HashKernel(n, seed=7)
    else:
        n = 10000
        k = core.ColorKernel(rng.random((n, 2)), 2)
    margs = [core.Histogram.normalized(rng.random(n) + 0.05) for _ in range(m)]
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    eng = B.BaryEngine(k, margs, np.full(m, 1.0 / m), prm)
    eng.load_state(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, fresh=True)
    for _ in range(3):
        eng.sweep()
        eng.update()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        eng.sweep()
        eng.update()
    e1.record(st)
    torch.cuda.synchronize()
    col = eng.col.cpu().numpy().copy()
    return e0.elapsed_time(e1) / iters, col


out = {}
for kind in ("stored", "points"):
    t2, c2 = run(kind, "1")
    t1, c1 = run(kind, "0")
    out[kind] = {"ms_per_iter_pairs": t2, "ms_per_iter_single": t1, "speedup": t1 / t2,
                 "max_rel_diff_cols": float(np.max(np.abs(c2 - c1)) / np.max(np.abs(c1)))}
    print(kind, json.dumps(out[kind]), flush=True)
