"""A/B timing of the single-read sweep vs the two-pass sweep (stored C, BASELINE config 3 shape).

    python tools/sr_bench.py [--n 100000] [--iters 10]

Times whole DXG iterations (sweep + O(n) update) with CUDA events on the launching stream,
from the bench's fresh state after 3 warm-up iterations per mode.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--modes", default="sr,two")
a = ap.parse_args()
n = a.n
rng = np.random.default_rng(1)
r, c = rng.random(n), rng.random(n)
r, c = r / r.sum(), c / c.sum()
k = core.HashKernel(n, seed=0)
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
st = torch.cuda.current_stream()
for mode in a.modes.split(","):
    sr = {"sr": True, "two": False}[mode]
    eng = DxgEngine(k, r, c, prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    for _ in range(3):
        eng.sweep(single_read=sr)
        eng.update()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(a.iters):
        eng.sweep(single_read=sr)
        eng.update()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    G = eng._sms()
    err = eng.slab.view(torch.int32)[2 * 16 * G * 8].item() if sr else 0
    print(f"{mode}: {ms:.3f} ms/iter  ({1e3 / ms:.2f} it/s, HBM one-read frac {8 * n * n / (ms * 1e-3) / 6552e9:.3f})"
          f"  wall {time.perf_counter() - t0:.2f}s err={err} a={eng.scal[0].item()}", flush=True)
    del eng
    torch.cuda.empty_cache()
