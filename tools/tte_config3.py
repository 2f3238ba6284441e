"""Config 3 (n=1e5 stored C, tuned+tau_mu=0.05) solved to eps (default 1e-4) within a wall-time bound.

Logs the solve trajectory (every log_stride iterations: primal, dual, gap, infeasibility,
seconds) through dxg.solve with a timeout, so time-to-eps can be read off (or
extrapolated) from real iterations on the benchmark instance.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--minutes", type=float, default=15.0)
ap.add_argument("--eps", type=float, default=1e-4)
ap.add_argument("--out", default="gpurun_out/tte_config3.json")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402

n = a.n
k = core.HashKernel(n, seed=0)
rng = np.random.default_rng(1)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
t0 = time.perf_counter()
sol = dxg.solve(k, core.Histogram(r), core.Histogram(c), prm,
                dxg.Termination(eps=a.eps, timeout=a.minutes * 60.0), log_stride=25, dense_cap=0)
wall = time.perf_counter() - t0
traj = [[p.iter, p.seconds, p.primal, p.dual, p.gap, p.col_infeas_l1] for p in sol.trajectory]
out = {"n": n, "eps": a.eps, "minutes_bound": a.minutes, "instance": "HashKernel(n, seed=0), marginals rng(1) as bench.py", "converged": sol.converged, "iterations": sol.iterations, "seconds": wall,
       "final": traj[-1], "trajectory_every_25": traj}
Path(a.out).write_text(json.dumps(out))
print(json.dumps({k2: v for k2, v in out.items() if k2 != "trajectory_every_25"}))
