"""Per-step timing of dxg.dxg_step from the zero state (fused vs two-pass diagnostics)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
k = core.HashKernel(n, seed=0)
rng = np.random.default_rng(1)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
st = dxg.DxgState(dxg.LogOddsField(np.zeros(n)), dxg.TransportLogWeights(0.0, np.zeros(n), 0.0, 0))
rh, ch = core.Histogram(r), core.Histogram(c)
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = dxg.dxg_step(st, k, rh, ch, prm)
    torch.cuda.synchronize()
    eng = dxg._STEP_CACHE["entry"]["eng"]
    print(i, f"{1e3 * (time.perf_counter() - t0):.1f} ms", "flags", eng.flags[0].item(), "a", st.weights.a,
          "nan(delta,b)", int(np.isnan(st.mu.delta).sum()), int(np.isnan(st.weights.b).sum()), flush=True)
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
for i in range(3):
    e0.record(); eng.sweep(); e1.record(); eng.update(); e2.record(); torch.cuda.synchronize()
    col = eng.col.cpu().numpy()
    print("sweep", e0.elapsed_time(e1), "update", e1.elapsed_time(e2), "col nan", int(np.isnan(col).sum()),
          "sums", col[:n].sum(), col[n:].sum(), flush=True)
