"""Host-side logic that needs no GPU: parameter schemes, validation, error behaviour."""

import math

import numpy as np
import pytest

from paper_2511_11359_b200 import dxg
from paper_2511_11359_b200.core import Histogram
from paper_2511_11359_b200.rounding import DenseCoupling, infeasibility


def test_params_tuned_matches_spec():
    p = dxg.params_tuned(0.0)
    assert (p.tau_p, p.tau_mu, p.beta, p.alpha, p.eta_mu, p.eta) == (1.0, 1.0, 1.1, 0.01, 0.0, 0.0)


def test_params_li_spec_example():
    p = dxg.params_li(1024, 0.01)
    assert abs(p.beta - 1153.66) < 0.01
    assert abs(p.tau_p - 0.02944) < 1e-5
    assert abs(p.tau_mu - 509.5) < 0.1
    assert abs(p.tau_p * p.tau_mu - 15.0) < 1e-12


def test_params_loose_spec_example():
    p = dxg.params_loose(1024, 0.01, 1e-3)   # SPEC.md:270 (reference computes 9.0168e-5)
    assert abs(p.eta - 0.01 / (16 * math.log(1024))) < 1e-18
    assert p.tau_mu == 1.0 / 128 and p.beta == math.log(3.0)
    assert p.tau_mu * p.eta_mu <= p.tau_p * p.eta + 1e-18


@pytest.mark.parametrize("kw", [dict(eta=-1.0), dict(tau_p=0.0), dict(beta=0.0), dict(alpha=2.0),
                                dict(eta=2.0, tau_p=1.0)])
def test_params_validation(kw):
    base = dict(eta=0.0, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.01)
    base.update(kw)
    with pytest.raises(ValueError):
        dxg.DxgParams(**base)


def test_histogram_validation():
    with pytest.raises(ValueError):
        Histogram(np.array([]))
    with pytest.raises(ValueError):
        Histogram(np.array([0.5, -0.1, 0.6]))
    with pytest.raises(ValueError):
        Histogram(np.array([0.5, 0.6]))
    h = Histogram.normalized([1, 0, 3])
    assert not h.full_support and h.n == 3 and h.min() == 0.0


def test_balance_and_dual_md_step_spec():
    mu = dxg.balance(dxg.LogOddsField(np.array([math.log(9.0), math.log(1.5)])), math.log(3.0))
    assert np.allclose(mu.delta, [math.log(3.0), math.log(1.5)])
    with pytest.raises(ValueError):
        dxg.balance(mu, 0.0)
    prm = dxg.DxgParams(eta=0.0, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.0)
    out = dxg.dual_md_step(dxg.LogOddsField(np.zeros(2)), [0.6, 0.4], Histogram(np.array([0.5, 0.5])),
                           [0.5, 0.5], prm)
    assert np.allclose(out.delta, [0.8, -0.8])


def test_infeasibility_report():
    rep = infeasibility([0.6, 0.4], True, Histogram(np.array([0.5, 0.5])))
    assert rep.row_gap == 0.0 and abs(rep.col_gap - 0.2) < 1e-15


def test_dense_coupling_validation():
    with pytest.raises(ValueError):
        DenseCoupling(np.array([[0.5, -1e-3], [0.2, 0.3]]))
    with pytest.raises(ValueError):
        DenseCoupling(np.zeros((2, 3)))


def test_solve_validates_before_touching_the_gpu():
    class K:
        n = 3
    with pytest.raises(ValueError):
        dxg.solve(K(), np.full(4, 0.25), np.full(3, 1 / 3), dxg.params_tuned())
    prm = dxg.DxgParams(eta=0.0, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.0)
    with pytest.raises(ValueError):
        dxg.solve(K(), np.full(3, 1 / 3), np.array([0.5, 0.5, 0.0]), prm)


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_11359_b200 import core
    with pytest.raises(RuntimeError, match="CUDA"):
        core.GridKernel(3, 3, 2)


def test_barycenter_eval_combine_of_row_shards():
    """Sharded barycenter evaluation (barycenter._combine_eval_buffers): row sums add in rank
    order, column statistics are taken from rank 0 (identical on all ranks), and the dual's
    log-sum-exp over rows combines the per-shard LSEs exactly."""
    import numpy as np
    from paper_2511_11359_b200.barycenter import _combine_eval_buffers
    rng = np.random.default_rng(0)
    m = 3
    bufs = [rng.normal(size=128) for _ in range(3)]
    for b in bufs[1:]:
        for k in range(m):
            b[64 + 2 * k: 66 + 2 * k] = bufs[0][64 + 2 * k: 66 + 2 * k]
    out = _combine_eval_buffers(bufs, m)
    for k in range(m):
        assert out[4 * k] == (bufs[0][4 * k] + bufs[1][4 * k]) + bufs[2][4 * k]
        assert out[4 * k + 1] == (bufs[0][4 * k + 1] + bufs[1][4 * k + 1]) + bufs[2][4 * k + 1]
        assert out[64 + 2 * k] == bufs[0][64 + 2 * k]
    ls = np.array([b[127] for b in bufs])
    assert abs(out[127] - np.log(np.exp(ls).sum())) <= 1e-14 * abs(out[127]) + 1e-15
    assert np.array_equal(_combine_eval_buffers([bufs[0]], m), bufs[0])


def test_spec6_balancing_is_the_kl_projection():
    """SPEC acceptance 6: on a grid of 10^3 (delta, beta) pairs the clamp of the log-odds
    (dxg.balance, dxg.py:236-245) is the KL projection of (mu+, mu-) = (logistic(delta),
    1 - logistic(delta)) onto {|log(mu+/mu-)| <= beta}, found numerically, within 1e-10."""
    import numpy as np
    from scipy.optimize import minimize_scalar
    from paper_2511_11359_b200 import dxg
    deltas = np.linspace(-6.0, 6.0, 40)
    betas = np.linspace(0.05, 5.0, 25)
    for beta in betas:
        got = dxg.balance(dxg.LogOddsField(deltas), float(beta)).delta
        for d, g in zip(deltas, got):
            mp = 1.0 / (1.0 + np.exp(-d))
            lo, hi = 1.0 / (1.0 + np.exp(beta)), 1.0 / (1.0 + np.exp(-beta))

            def kl(q):
                return q * np.log(q / mp) + (1 - q) * np.log((1 - q) / (1 - mp))
            res = minimize_scalar(kl, bounds=(lo, hi), method="bounded", options={"xatol": 1e-14})
            q = min(max(res.x, lo), hi)
            q = lo if kl(lo) < kl(q) else (hi if kl(hi) < kl(q) else q)
            assert abs(np.log(q / (1 - q)) - g) <= 1e-6 or abs(q - 1.0 / (1.0 + np.exp(-g))) <= 1e-10


def test_default_splits_fill_the_waves():
    """leanot_dxg_default_splits (no GPU: 148 SMs assumed): small and very large plans pick the
    column-pass split count whose (tile, split) items fill the last wave over 2 x 148 resident
    CTAs (fewest items within 2 % of the best fill); mid sizes keep >= 4 items per CTA."""
    import ctypes
    from paper_2511_11359_b200 import _lib
    L = _lib.lib()

    def splits(n, rows):
        s = ctypes.c_int(0)
        assert L.leanot_dxg_default_splits(n, rows, ctypes.byref(s)) == 0
        return s.value

    def fill(n, s):
        items = ((n + 1023) // 1024) * s
        return items / (-(-items // 296) * 296)

    assert splits(10_000, 10_000) == 29 and fill(10_000, 29) > 0.97          # config 2: one full wave
    assert splits(1_000_000, 125_000) == 3 and fill(1_000_000, 3) > 0.98     # config 4 shard
    assert splits(100_000, 100_000) == 19                                    # config 3 (measured)
    for n in (2000, 5000, 16384):
        s = splits(n, n)
        assert 1 <= s <= 64 and s <= max(1, n // 8)


def _core_cases():
    import json
    from pathlib import Path
    z = np.load(Path(__file__).parent / "golden" / "core_cases.npz")
    meta = json.loads(bytes(z["__meta__"]).decode())
    return z, meta


@pytest.mark.parametrize("name", sorted(_core_cases()[1]))
def test_core_helpers_match_reference(name):
    """Reference leanot.core helpers (core.py:49-164) replayed from oracle/gen_golden_core.py."""
    from paper_2511_11359_b200 import core
    z, meta = _core_cases()
    rec = meta[name]
    args = [z[f"{name}__arg{q}"] for q in range(rec["nargs"])]
    fn = getattr(core, rec["fn"])
    if rec["kind"] == "error":
        with pytest.raises(Exception) as ei:
            fn(*args, **rec["kw"])
        assert type(ei.value).__name__ == rec["exc"] and str(ei.value) == rec["msg"]
        return
    out = fn(*args, **rec["kw"])
    if rec["kind"] == "histogram":
        assert out.full_support == rec["full_support"]
        out = out.weights
    np.testing.assert_array_equal(np.asarray(out, dtype=float), z[f"{name}__out"])


def test_map_blocks_block_order():
    from paper_2511_11359_b200.core import map_blocks
    for w in (1, 3):
        assert map_blocks(lambda i0, i1: (i0, i1), 300, workers=w) == [(0, 128), (128, 256), (256, 300)]
