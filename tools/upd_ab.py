"""Per-iteration time of the regular engine path and of graph-replayed iterations at size n
(A/B of the O(n) update variants via LEANOT_SMALL_UPD_N)."""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--kind", default="points2")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

n = a.n
rng = np.random.default_rng(2)
k = core.ColorKernel(rng.random((n, 2)), 2) if a.kind == "points2" else core.ExplicitKernel(rng.random((n, n)))
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
eng = DxgEngine(k, r, c, dxg.params_tuned(1e-6).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
st = torch.cuda.current_stream()


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


def step():
    eng.sweep(); eng.update()


def upd():
    eng.update()


timed(step, 20)
t_step = timed(step, 200) / 200
t_upd = timed(upd, 200) / 200
eng.iterate(25)
torch.cuda.synchronize()
t_graph = timed(lambda: eng.iterate(25), 8) / 200
print(json.dumps({"n": n, "kind": a.kind, "small_upd_n": os.environ.get("LEANOT_SMALL_UPD_N", "default"),
                  "us_per_iter": t_step, "us_update_only": t_upd, "us_per_iter_graph": t_graph}))
