"""A few separable-path iterations for ncu launch lists: config-5 barycenter (m=8) or one DXG grid sweep."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path[:0] = [str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parent)]
ap = argparse.ArgumentParser()
ap.add_argument("--what", default="bary", choices=["bary", "dxg"])
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import barycenter as B  # noqa: E402
from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

side, m = 316, 8
n = side * side
rng = np.random.default_rng(5)
g = core.GridKernel(side, side, 2)
prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
if a.what == "bary":
    margs = [core.Histogram.normalized(rng.random(n)) for _ in range(m)]
    eng = B.BaryEngine(g, margs, np.full(m, 1.0 / m), prm)
    eng.load_state(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, fresh=True)
else:
    r = rng.random(n); r /= r.sum()
    c = rng.random(n); c /= c.sum()
    eng = DxgEngine(g, r, c, prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
for _ in range(2 + a.iters):
    eng.sweep(); eng.update()
torch.cuda.synchronize()
