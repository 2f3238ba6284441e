"""Fused single-launch sweep (stored cost, csrc/leanot_fused.cu) vs the two-pass sweep (needs a B200).

With LEANOT_SWEEP_FUSED (engine.sweep(fused=True)) a plain DXG iteration sweep of a stored
cost with even n >= 16384 runs as one persistent kernel (pass B trails pass A by two
16-row panels and re-reads C from L2).  It is opt-in (slower than the two-pass kernels as
of r01), and must give the same iteration: both are compared on the same
state -- column marginals, row outputs and whole iterations.
Tolerance: the two forms sum the same terms in different orders (fixed in each), so they
agree to a few ulps of the sums -- checked at 1e-13 relative (north_star: 1e-10).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


def _setup(n, a, seed, rows=None):
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(seed)
    k = core.HashKernel(n, seed=seed, rows=rows) if rows else core.HashKernel(n, seed=seed)
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 0.05 * a, n))
    b -= b.max()
    return k, r, c, prm, (delta, b, a, 0.2, 100)


def _two_pass(eng):
    eng.sweep_phase("rows")
    eng.sweep_phase("cols")


@pytest.mark.parametrize("n,a", [(16384, 40.0), (20002, 800.0), (30000, 5000.0)])
def test_fused_sweep_matches_two_pass(n, a):
    import torch
    from paper_2511_11359_b200.engine import DxgEngine
    k, r, c, prm, st = _setup(n, a, n)
    out = []
    for fused in (True, False):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(*st)
        eng.sweep(fused=True) if fused else _two_pass(eng)
        torch.cuda.synchronize()
        if fused:  # the fused kernel ran: panel 0's arrival counter (after the partial-sum slots) == units
            G = eng._sms()
            q = G // 4
            part_d = 8 * 16 * 2 * q
            assert eng.slab.view(torch.int32)[2 * part_d].item() == 4 * q
        out.append((eng.col.cpu().numpy().copy(), eng.S.cpu().numpy().copy(), eng.shift.cpu().numpy().copy(),
                    eng.flags[0].item()))
        del eng
    (c0, s0, h0, f0), (c1, s1, h1, f1) = out
    assert f0 == 0 and f1 == 0
    assert rel_err(c0[:n], c1[:n]) <= 1e-13 and rel_err(c0[n:], c1[n:]) <= 1e-13
    assert abs(c0[:n].sum() - 1.0) <= 1e-12 and abs(c0[n:].sum() - 1.0) <= 1e-12
    assert rel_err(s0, s1) <= 1e-13
    assert np.array_equal(h0, h1) or np.max(np.abs(h0 - h1)) <= 1    # next shifts (llrint of log S)


def test_fused_iterations_track_two_pass():
    from paper_2511_11359_b200.engine import DxgEngine
    n = 20000
    k, r, c, prm, st = _setup(n, 300.0, 5)
    states = []
    for fused in (True, False):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(*st)
        for _ in range(25):
            eng.sweep(fused=True) if fused else _two_pass(eng)
            eng.update()
        states.append(eng.read_state())
    (d0, b0, a0, s0, t0), (d1, b1, a1, s1, t1) = states
    assert rel_err(d0, d1) <= 1e-11 and rel_err(b0, b1) <= 1e-11
    assert a0 == a1 and s0 == s1 and t0 == t1 == 125


def test_fused_sweep_is_deterministic_and_covers_row_shards():
    import torch
    from paper_2511_11359_b200.engine import DxgEngine
    n = 24000
    k, r, c, prm, st = _setup(n, 900.0, 11)
    eng = DxgEngine(k, r, c, prm)
    eng.load_state(*st)
    sh = eng.shift.clone()
    eng.sweep(fused=True)
    a = eng.col.clone()
    eng.shift.copy_(sh)
    eng.sweep(fused=True)
    assert torch.equal(a, eng.col)
    # row shard [5000, 17013): fused partial == two-pass partial
    ks, r2, c2, prm2, st2 = _setup(n, 900.0, 11, rows=(5000, 17013))
    out = []
    for fused in (True, False):
        e = DxgEngine(ks, r2, c2, prm2)
        assert (e.row0, e.row1) == (5000, 17013)
        e.load_state(*st2)
        e.sweep(fused=True) if fused else _two_pass(e)
        out.append(e.col.cpu().numpy().copy())
    assert rel_err(out[0], out[1]) <= 1e-13


def test_fused_fixup_of_flagged_rows():
    """A jump in a makes every row's shift wrong by ~1e3 (row sums far outside [2^-900, 2^900]):
    pass B skips the rows, fused_fix_kernel recomputes them exactly and adds their columns."""
    import torch
    from paper_2511_11359_b200.engine import DxgEngine
    n = 16384
    k, r, c, prm, st = _setup(n, 10.0, 3)
    out = []
    for fused in (True, False):
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(*st)
        eng.scal[0] = 3000.0
        eng.scal[1] = 3000.5
        eng.sweep(fused=True) if fused else _two_pass(eng)
        torch.cuda.synchronize()
        out.append((eng.col.cpu().numpy().copy(), eng.flags[0].item()))
    (c0, f0), (c1, f1) = out
    assert f0 == 0 and f1 == 0                  # fixup lists consumed
    assert np.all(np.isfinite(c0))
    assert rel_err(c0, c1) <= 1e-12
