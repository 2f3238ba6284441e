"""Time pass A / pass B / update of the DXG engine at size n (CUDA events, median of K)."""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--kind", default="hash")
ap.add_argument("--tag", default="")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

n = a.n
rng = np.random.default_rng(1)
if a.kind == "hash":
    k = core.HashKernel(n, seed=0)
elif a.kind == "points2":
    k = core.ColorKernel(rng.random((n, 2)), 2, scale=2.0)
elif a.kind == "points3":
    k = core.ColorKernel(rng.random((n, 3)), 2, scale=3.0)
else:
    side = int(round(n ** 0.5))
    k = core.GridKernel(side, side, 2)
    n = k.n
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
for _ in range(3):
    eng.sweep(); eng.update()
torch.cuda.synchronize()
import subprocess  # noqa: E402
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "100"], stdout=subprocess.PIPE, text=True)
st = torch.cuda.current_stream()
ta, tb = [], []
for _ in range(a.iters):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st); eng.sweep_phase("rows"); e[1].record(st); eng.sweep_phase("cols"); e[2].record(st)
    eng.update()
    torch.cuda.synchronize()
    ta.append(e[0].elapsed_time(e[1])); tb.append(e[1].elapsed_time(e[2]))
smi.terminate()
rows = [line.split(",") for line in smi.stdout.read().splitlines() if line.strip()]
clk = [float(x[0]) for x in rows]
pw = [float(x[1]) for x in rows]
print(json.dumps({"tag": a.tag, "n": n, "kind": a.kind, "rowpass_ms": statistics.median(ta),
                  "colpass_ms": statistics.median(tb), "sm_mhz": statistics.median(clk) if clk else None,
                  "power_w": statistics.median(pw) if pw else None}))
