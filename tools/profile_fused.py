"""A few fused DXG sweeps (stored cost) at size n, for ncu captures of fused_sweep_kernel."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
k = core.HashKernel(n, seed=0)
rng = np.random.default_rng(1)
r = rng.random(n); r /= r.sum()
c = rng.random(n); c /= c.sum()
eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(4):
    e0.record(); eng.sweep(fused=True); e1.record(); eng.update(); torch.cuda.synchronize()
    print("fused sweep ms", e0.elapsed_time(e1), flush=True)
for i in range(2):
    e0.record(); eng.sweep_phase("rows"); eng.sweep_phase("cols"); e1.record(); eng.update(); torch.cuda.synchronize()
    print("two-pass sweep ms", e0.elapsed_time(e1), flush=True)
