"""Config-3 time to eps across several bounded GPU sessions (checkpoint / resume).

    python tools/tte_resume.py --eps 1e-5 --minutes 50 --ckpt ckpt/tte.npz --out gpurun_out/tte_seg.npz

A gpurun call lasts at most one hour, fewer than a run to eps = 1e-5 needs, so this runs
the solve loop of dxg.solve (dxg.py:420-472: iterations between logging points without host
syncs, an evaluation sweep every log_stride iterations that doubles as the next sweep,
gap <= eps/6 and infeasibility <= eps/6) for a wall-time budget, then writes the state
(delta, b, a, s, t), the accumulated trajectory and the accumulated solve seconds.  The next
session resumes from that file.  On resume the row shifts are recomputed from exact row
maxima (load_state), which changes the summation path by ~1e-15 relative; in the
tuned + tau_mu = 0.05 regime this is far below the iteration's sensitivity.
Seconds are summed solve time (setup of each session excluded).
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--eps", type=float, default=1e-5)
ap.add_argument("--minutes", type=float, default=50.0)
ap.add_argument("--ckpt", default="")
ap.add_argument("--out", required=True)
ap.add_argument("--log-stride", type=int, default=25)
a = ap.parse_args()

n = a.n
k = core.HashKernel(n, seed=0)
rng = np.random.default_rng(1)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
eng = DxgEngine(k, r, c, prm)
if a.ckpt and Path(a.ckpt).exists():
    z = np.load(a.ckpt)
    it = int(z["t"])
    eng.load_state(z["delta"], z["b"], float(z["a"]), float(z["s"]), it)
    traj = [list(x) for x in z["traj"]]
    secs0 = float(z["seconds"])
    segments = int(z["segments"]) + 1
else:
    it = 0
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    traj, secs0, segments = [], 0.0, 1
torch.cuda.synchronize()
t0 = time.perf_counter()
budget = a.minutes * 60.0
swept = False
converged = False
stride = a.log_stride
while time.perf_counter() - t0 < budget:
    nxt = ((it // stride) + 1) * stride
    if not swept:
        eng.sweep()
    eng.update()
    eng.iterate(nxt - it - 1)
    it = nxt
    eng.sweep(evaluate=True)
    swept = True
    primal, dual, infeas = eng.evaluate()        # one device->host read per logging point
    s_val = eng.last_scalars[2]
    traj.append([it, secs0 + time.perf_counter() - t0, primal, dual, primal - dual, infeas, s_val])
    if primal - dual <= a.eps / 6.0 and infeas <= a.eps / 6.0:
        converged = True
        break
seconds = secs0 + time.perf_counter() - t0
delta, b, av, sv, tv = eng.read_state()
assert tv == it, (tv, it)
np.savez(a.out, delta=delta, b=b, a=av, s=sv, t=it, traj=np.array(traj), seconds=seconds, segments=segments,
         converged=converged, eps=a.eps)
print({"iterations": it, "converged": converged, "seconds": seconds, "segments": segments,
       "last": traj[-1] if traj else None}, flush=True)
