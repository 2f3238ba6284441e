"""Pass-B time vs the number of row splits (wave quantization of the column pass)."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
splits_list = [int(x) for x in sys.argv[3].split(",")]
rng = np.random.default_rng(1)
if kind == "hash":
    k = core.HashKernel(n, seed=0)
elif kind == "points3shard":   # BASELINE config 4: a 1/8 row shard of n 3-D points
    k = core.ColorKernel(rng.random((n, 3)), 2, scale=3.0)
    k.row0, k.row1 = 0, n // 8
else:
    k = core.ColorKernel(rng.random((n, 2)), 2, scale=2.0)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
for s in splits_list:
    eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05), splits=s)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    for _ in range(3):
        eng.sweep(); eng.update()
    tb = []
    reps = 3 if n >= 50000 else 50
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); eng.sweep_phase("rows"); e[1].record(); eng.sweep_phase("cols"); e[2].record()
        eng.update(); torch.cuda.synchronize()
        tb.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
    print(json.dumps({"kind": kind, "n": n, "splits": s, "rowpass_ms": statistics.median(x[0] for x in tb),
                      "colpass_ms": statistics.median(x[1] for x in tb)}), flush=True)
    del eng
    torch.cuda.empty_cache()
