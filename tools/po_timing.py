"""Phase timestamps of the row-owner persistent kernel (library built with -DLEANOT_DBG_TIMING)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)
r = core.Histogram.normalized(rng.random(n)).weights
c = core.Histogram.normalized(rng.random(n)).weights
k = core.ExplicitKernel(rng.random((n, n)))
eng = DxgEngine(k, r, c, dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
for _ in range(3):
    eng.iterate(10)
    torch.cuda.synchronize()
    ts = eng.partial[:8].view(torch.int64).cpu().numpy()
    print("phase ns:", np.diff(ts).tolist(), "total", ts[7] - ts[0])
