"""Shared test helpers: golden fixtures and kernel construction from fixture arrays."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    d = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return {k: d[k] for k in d.files}


def meta(d):
    return json.loads(str(d["meta"]))


def golden_names(prefix):
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


def kind_of(d):
    if "kind" in d:
        return str(d["kind"])
    return meta(d)["kind"]


def oracle_cost(d):
    import leanot_oracle as O
    kind = kind_of(d)
    if kind == "explicit":
        return O.DenseCost(d["k_C"])
    if kind == "grid":
        return O.GridCost(int(d["k_H"]), int(d["k_W"]), int(d["k_p"]))
    return O.PointCost(d["k_F"], int(d["k_p"]))


def device_cost(d):
    from paper_2511_11359_b200 import core
    kind = kind_of(d)
    if kind == "explicit":
        return core.ExplicitKernel(d["k_C"])
    if kind == "grid":
        return core.GridKernel(int(d["k_H"]), int(d["k_W"]), int(d["k_p"]))
    return core.ColorKernel(d["k_F"], int(d["k_p"]))


def rel_err(x, ref):
    x, ref = np.asarray(x, dtype=float), np.asarray(ref, dtype=float)
    scale = max(float(np.max(np.abs(ref))), 1e-300)
    return float(np.max(np.abs(x - ref))) / scale


def params_from(arr):
    import leanot_oracle as O
    eta, eta_mu, tau_p, tau_mu, beta, alpha = (float(v) for v in arr)
    return O.Params(eta, eta_mu, tau_p, tau_mu, beta, alpha)
