"""Run DXG sweeps back to back for a few seconds and sample SM clock, power and throttle reasons.

Tells whether the sweep kernels are held below max clock by the power limit (and which one).
"""
import argparse
import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--seconds", type=float, default=4.0)
ap.add_argument("--phase", default="both", choices=["both", "rows", "cols"])
a = ap.parse_args()
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

fields = ("clocks.sm,clocks.max.sm,power.draw,power.draw.instant,enforced.power.limit,power.max_limit,"
          "temperature.gpu,clocks_event_reasons.active")
static = subprocess.run(["nvidia-smi", "--query-gpu=" + fields, "--format=csv"], capture_output=True, text=True).stdout
n = a.n
rng = np.random.default_rng(1)
k = core.HashKernel(n, seed=0)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
for _ in range(3):
    eng.sweep(); eng.update()
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=" + fields, "--format=csv,noheader,nounits", "-lms", "50"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
t0 = time.time()
iters = 0
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
while time.time() - t0 < a.seconds:
    for _ in range(10):
        if a.phase == "both":
            eng.sweep(); eng.update()
        else:
            eng.sweep_phase(a.phase)
        iters += 1
    torch.cuda.synchronize()
e1.record(st)
torch.cuda.synchronize()
smi.terminate()
rows = [x.split(", ") for x in smi.stdout.read().splitlines() if x.strip()]
print(static.strip())
for x in rows[:: max(1, len(rows) // 25)]:
    print(", ".join(x))
print(json.dumps({"phase": a.phase, "iters": iters, "ms_per_iter": e0.elapsed_time(e1) / iters}))
