"""Quick correctness probe of the TMA-staged stored-cost sweeps vs the oracle (even n)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import leanot_oracle as O  # noqa: E402

from paper_2511_11359_b200 import core, dxg  # noqa: E402

for n in (2, 10, 1000, 2048, 3000, 4100):
    rng = np.random.default_rng(n)
    Cm = rng.random((n, n))
    r = O.normalized_hist(rng.random(n))
    k = core.ExplicitKernel(Cm, cap=None)
    a, b = 37.0, -np.abs(rng.normal(0, 5, n))
    col = dxg.column_marginal(dxg.TransportLogWeights(a, b, 0, 0), k, r)
    (ref,) = O.column_marginals(O.DenseCost(Cm), r, [(a, b)])
    err = np.max(np.abs(col - ref)) / np.max(np.abs(ref))
    print(n, f"{err:.2e}")
    assert err < 1e-12, n
print("tma smoke ok")
