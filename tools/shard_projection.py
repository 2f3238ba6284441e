"""Per-rank work of the row-sharded config-3 iteration, measured on one GPU.

For N in {1, 2, 4, 8}: rank 0's shard of BASELINE config 3 (n = 1e5 stored C, rows
[0, n/N)) is swept and updated exactly as in a multi-GPU run (leanot_dxg_sweep on the
shard, the O(n) update on all columns); the NCCL exchange (all-gather of N x 2n doubles,
rank-order sum) is not included -- it is ~1-2e-5 s per iteration on NVLink 5 (12.8 MB at
N = 8).  Prints the per-iteration shard time and the implied iterations/s.
"""
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine, shard_rows  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
rng = np.random.default_rng(1)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
for N in (1, 2, 4, 8):
    r0, r1 = shard_rows(n, N, 0)
    k = core.HashKernel(n, seed=0, rows=(r0, r1))
    eng = DxgEngine(k, r, c, prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    for _ in range(3):
        eng.sweep(); eng.update()
    ts = []
    for _ in range(6 if N < 4 else 12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eng.sweep(); eng.update(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.median(ts)
    print(json.dumps({"N": N, "rows": r1 - r0, "seconds_per_iter": t, "iters_per_s_projected": 1.0 / t}), flush=True)
    del eng, k
    torch.cuda.empty_cache()
