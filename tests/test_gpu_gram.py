"""Expanded (Gram) form of squared-Euclidean point costs vs the difference form (needs a B200).

ColorKernel with p = 2 carries |f_j|^2 (leanot_cost_t.norms); the plain DXG iteration
sweeps then evaluate a C_ij through a inv (N_i + N_j - 2 f_i.f_j) with the row term
dropped (it cancels in the row softmax, dxg.py:199-202).  The same kernel object with
the norms removed runs the difference form sum_d (f_id - f_jd)^2 of the reference
(core.py:264-288).  Both must give the same iteration to the north_star tolerance
(1e-10 relative per iteration), including states far from the initial one (large a,
where the expanded form's cancellation is largest).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


def _pair(n, d, seed, offset=0.0):
    from paper_2511_11359_b200 import core
    rng = np.random.default_rng(seed)
    f = rng.random((n, d)) + offset
    kg = core.ColorKernel(f, 2)
    kd = core.ColorKernel(f, 2, scale=kg.scale)
    kd.norms_dev = None            # difference form
    assert kg.norms_dev is not None and kg.cost_struct().norms and not kd.cost_struct().norms
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    return kg, kd, r, c, rng


@pytest.mark.parametrize("n,d,a,offset", [(5001, 2, 40.0, 0.0), (20000, 3, 5000.0, 0.0), (4097, 1, 800.0, 0.0),
                                          (6000, 4, 200.0, 0.0), (8000, 3, 2000.0, 1000.0), (3001, 2, 300.0, -250.0)])
def test_gram_iterations_track_difference_form(n, d, a, offset):
    """offset != 0: point clouds far from the origin (the expanded form runs on centered
    features, so its cancellation error does not grow with |f|^2)."""
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200.engine import DxgEngine
    kg, kd, r, c, rng = _pair(n, d, n + d, offset)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 0.05 * a, n))
    b -= b.max()
    cols, states = [], []
    for k in (kg, kd):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(delta, b, a, 0.0, 100)
        eng.sweep()
        cols.append(eng.col.cpu().numpy().copy())
        eng.update()
        eng.iterate(20, use_graph=False)
        states.append(eng.read_state())
    assert rel_err(cols[0][:n], cols[1][:n]) <= 1e-11
    assert rel_err(cols[0][n:], cols[1][n:]) <= 1e-11
    (d0, b0, a0, s0, t0), (d1, b1, a1, s1, t1) = states
    assert rel_err(d0, d1) <= 1e-10 and rel_err(b0, b1) <= 1e-10
    assert a0 == a1 and s0 == s1 and t0 == t1 == 121


def test_gram_row_fixup_path():
    """Shifts far from the row normalizers (a jump in a between load and sweep) force the exact
    recompute of flagged rows; the expanded form must convert its shifts consistently."""
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n = 3000
    kg, kd, r, c, rng = _pair(n, 3, 7)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 20, n))
    b -= b.max()
    out = []
    for k in (kg, kd):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(delta, b, 10.0, 0.0, 100)           # exact row maxima for a = 10
        eng.scal[0] = 3000.0                                # a jumps: shifts are off by ~1e3
        eng.scal[1] = 3000.5
        eng.sweep()
        out.append(eng.col.cpu().numpy().copy())
    assert np.all(np.isfinite(out[0]))
    assert rel_err(out[0], out[1]) <= 1e-11
