"""A few single-read sweeps on a row shard of the n = 1e5 hash matrix, for ncu captures of
sr_sweep_kernel (stored C, BASELINE config 3 shape; the shard keeps ncu's replays short).

    python tools/profile_sr.py [--n 100000] [--rows 16000] [--reps 3]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--rows", type=int, default=16000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = a.n
rng = np.random.default_rng(1)
r, c = rng.random(n), rng.random(n)
k = core.HashKernel(n, seed=0, rows=(0, a.rows))
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
eng = DxgEngine(k, r / r.sum(), c / c.sum(), prm)
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(a.reps):
    e0.record()
    eng.sweep(single_read=True)
    e1.record()
    eng.update()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"sr sweep {ms:.3f} ms for {a.rows} rows: {ms * 1e3 / ((a.rows + 3) // 4):.3f} us/panel", flush=True)
