"""Golden cases for the reference's O(n) core helpers, produced by running the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_core.py

Feeds seeded inputs (and the error cases) to leanot.core's ingest_image_histogram, lse,
lse_rows, kl_divergence, entropy and logistic (core.py:49-164) and records the reference's
output or the exception it raised in tests/golden/core_cases.npz.  tests/test_host_logic.py
replays them against paper_2511_11359_b200.core (test infrastructure; the reference does
not travel).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from leanot import core as RC  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "core_cases.npz"


def cases():
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=(7, 9)).astype(float)
    img_zeros = img.copy()
    img_zeros[0, :4] = 0.0
    yield "ingest", "ingest_image_histogram", (img,), {}
    yield "ingest_p0", "ingest_image_histogram", (img_zeros,), {"perturbation": 0.0}
    yield "ingest_p1e-3", "ingest_image_histogram", (img_zeros,), {"perturbation": 1e-3}
    yield "ingest_neg", "ingest_image_histogram", (np.array([[1.0, -1.0]]),), {}
    yield "ingest_zero", "ingest_image_histogram", (np.zeros((2, 2)),), {}
    v = rng.normal(size=50) * 30
    yield "lse", "lse", (v,), {}
    yield "lse_neginf", "lse", (np.array([-np.inf, 1.0, 2.0]),), {}
    yield "lse_allneginf", "lse", (np.array([-np.inf, -np.inf]),), {}
    yield "lse_empty", "lse", (np.array([]),), {}
    yield "lse_nan", "lse", (np.array([1.0, np.nan]),), {}
    yield "lse_rows", "lse_rows", (rng.normal(size=(6, 11)) * 50,), {}
    a = rng.random(40)
    a /= a.sum()
    b = rng.random(40)
    b /= b.sum()
    a0 = a.copy()
    a0[:5] = 0.0
    yield "kl", "kl_divergence", (a, b), {}
    yield "kl_zeros", "kl_divergence", (a0, b), {}
    b0 = b.copy()
    b0[3] = 0.0
    yield "kl_not_ac", "kl_divergence", (a, b0), {}
    yield "kl_shape", "kl_divergence", (a, b[:-1]), {}
    yield "entropy", "entropy", (a0,), {}
    yield "logistic", "logistic", (rng.normal(size=64) * 400,), {}


def main():
    arrays, meta = {}, {}
    for name, fn, args, kw in cases():
        for q, x in enumerate(args):
            arrays[f"{name}__arg{q}"] = np.asarray(x, dtype=float)
        rec = {"fn": fn, "nargs": len(args), "kw": kw}
        try:
            out = getattr(RC, fn)(*args, **kw)
            if isinstance(out, RC.Histogram):
                arrays[f"{name}__out"] = out.weights
                rec["full_support"] = bool(out.full_support)
                rec["kind"] = "histogram"
            else:
                arrays[f"{name}__out"] = np.asarray(out, dtype=float)
                rec["kind"] = "array"
        except Exception as e:  # recorded, replayed as the same exception type + message
            rec["kind"] = "error"
            rec["exc"] = type(e).__name__
            rec["msg"] = str(e)
        meta[name] = rec
    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({len(meta)} cases)")


if __name__ == "__main__":
    main()
