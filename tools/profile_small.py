"""A few DXG iterations at small n (BASELINE config 1 shape) for launch lists."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

rng = np.random.default_rng(0)
n = a.n
r = core.Histogram.normalized(rng.random(n)).weights
c = core.Histogram.normalized(rng.random(n)).weights
k = core.ExplicitKernel(rng.random((n, n)))
eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
eng.iterate(a.iters, use_graph=bool(a.graph))
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
eng.iterate(200, use_graph=True)
torch.cuda.synchronize()
e0.record(st)
eng.iterate(200, use_graph=True)
e1.record(st)
torch.cuda.synchronize()
print("us per iteration (graph of 200):", e0.elapsed_time(e1) * 1e3 / 200)
for chunk in (24, 200):
    eng.iterate(chunk, use_graph=False)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(200 // chunk):
        eng.iterate(chunk, use_graph=False)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"us per iteration (leanot_dxg_iterate, chunks of {chunk}):", e0.elapsed_time(e1) * 1e3 / (chunk * (200 // chunk)))
