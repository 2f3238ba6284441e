"""Fixtures for the SPEC acceptance criteria that need the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python oracle/gen_golden_spec.py

Writes tests/golden/spec_acceptance.npz:
  * criterion 1 (PDXG <-> DXG): the reference's dense PDXG iterate (`pdxg_reference_step`,
    dxg.py:494-521) after 500 loose-parameter iterations for n in {4, 8, 16} (one seed each),
    which pins the oracle's restatement (`leanot_oracle.pdxg_step`) that the GPU test then
    runs for all 20 seeds;
  * criterion 4 (OT optimality): the exact transport LP value (`oracle.exact_ot`,
    oracle.py:149-192) of 8x8 grid instances, p in {1, 2}, in normalized cost units.
Test infrastructure only; the reference is not available on the GPU box.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from leanot import core, dxg  # noqa: E402
from leanot import oracle as LP  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "spec_acceptance.npz"


def pdxg_case(n: int, seed: int):
    rng = np.random.default_rng(1000 + seed)
    C = rng.random((n, n))
    r = core.Histogram.normalized(rng.random(n) + 0.1)
    c = core.Histogram.normalized(rng.random(n) + 0.1)
    k = core.ExplicitKernel(C)
    prm = dxg.params_loose(n, 1e-2, float(c.weights.min()), k.sup_norm)
    st = dxg.pdxg_init(n)
    for _ in range(500):
        st = dxg.pdxg_reference_step(st, k, r, c, prm)
    return C, r.weights, c.weights, prm, st


def main():
    arrays = {}
    for n in (4, 8, 16):
        C, r, c, prm, st = pdxg_case(n, 0)
        arrays[f"pdxg{n}_C"] = C
        arrays[f"pdxg{n}_r"] = r
        arrays[f"pdxg{n}_c"] = c
        arrays[f"pdxg{n}_params"] = np.array([prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha])
        arrays[f"pdxg{n}_log_p"] = st.log_p
        arrays[f"pdxg{n}_delta"] = st.mu.delta
    for p in (1, 2):
        rng = np.random.default_rng(40 + p)
        k = core.GridKernel(8, 8, p)
        r = core.Histogram.normalized(rng.random(64) + 0.05)
        c = core.Histogram.normalized(rng.random(64) + 0.05)
        sol = LP.exact_ot(k, r, c)
        arrays[f"lp{p}_r"] = r.weights
        arrays[f"lp{p}_c"] = c.weights
        arrays[f"lp{p}_value"] = np.array(sol.value)
        arrays[f"lp{p}_dual"] = np.array(sol.dual_value(r, c))
    arrays["meta"] = np.array(json.dumps({"numpy": np.__version__, "block_rows": core.BLOCK_ROWS,
                                          "pdxg_iterations": 500, "pdxg_params": "params_loose(n, 1e-2, min c)",
                                          "lp": "8x8 GridKernel, exact_ot value (normalized costs)"}))
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT, sorted(arrays))


if __name__ == "__main__":
    main()
