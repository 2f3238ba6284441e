"""Parity at BASELINE.json's full sizes through size-independent properties (needs a B200).

The oracle cannot sweep n = 1e5 x 1e5 (config 3) or a 1e6-point shard (config 4)
in test time, so at those sizes the CUDA path is checked through properties
that hold for any n:

  * row-block decomposition: the column partial of any row block equals the
    oracle's r_blk @ softmax(-(a C_blk + b)) over ALL n columns
    (dxg.py:199-203), for sampled blocks at the start, middle and end;
  * mass conservation: sum_j col_j == sum_i r_i for both half-step weight sets;
  * O(n) update: the GPU's next state equals the oracle's dual_md_step /
    _advance_weights (dxg.py:223-258) applied to the GPU's own columns;
  * determinism: two sweeps of the same state (same row shifts) are bitwise identical;
  * shard additivity: row-shard partials summed in rank order equal
    the unsharded columns (engine.combine_partials, multi-GPU path).
"""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu

TOL_BLOCK = 1e-12     # partial columns of a row block vs the oracle (1e5 / 1e6 terms per row)
TOL_MASS = 1e-13
TOL_UPDATE = 1e-13


def _hist(rng, n):
    w = rng.random(n)
    return w / w.sum()


def _state(rng, n, a):
    delta = rng.uniform(-2.0, 2.0, n)
    b = -np.abs(rng.normal(0.0, 0.05 * a, n))
    b -= b.max()
    return delta, b, float(a), 0.3, 100


def _engine(kernel, r, c, prm, st):
    from paper_2511_11359_b200.engine import DxgEngine
    eng = DxgEngine(kernel, r, c, prm)
    eng.load_state(*st)
    return eng


def _cols(eng):
    eng.sweep()
    col = eng.col.cpu().numpy()
    return col[: eng.n].copy(), col[eng.n:].copy()


def _bar_weights(st, prm, sup):
    delta, b, a, s, t = st
    a_bar, b_bar, _, _ = O._advance(a, b, s, t, np.tanh(0.5 * delta), prm, sup)
    return a_bar, b_bar


def _oracle_block(cost_block, r, weight_sets, i0, i1):
    return [r[i0:i1] @ O._softmax_block(a, b, cost_block) for a, b in weight_sets]


def _oracle_prm():
    return O.params_tuned(0.0, tau_mu=0.05)


def _release():
    import gc

    import torch
    gc.collect()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("a", [500.0, 5000.0])
def test_config3_full_size_properties(a):
    """BASELINE config 3: n = 1e5, stored C (80 GB in HBM)."""
    from paper_2511_11359_b200 import core, dxg
    n = 100_000
    rng = np.random.default_rng(int(a))
    r, c = _hist(rng, n), _hist(rng, n)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    oprm = _oracle_prm()
    st = _state(rng, n, a)
    hc = O.HashCost(n, seed=7)
    ws = [(st[2], st[1]), _bar_weights(st, oprm, 1.0)]
    try:
        k = core.HashKernel(n, seed=7)
        eng = _engine(k, r, c, prm, st)
        col_now, col_bar = _cols(eng)
        eng.load_state(*st)             # same state, same (exact row-max) shifts
        again = _cols(eng)
        assert np.array_equal(col_now, again[0]) and np.array_equal(col_bar, again[1])   # deterministic
        for col in (col_now, col_bar):
            assert abs(col.sum() - r.sum()) <= TOL_MASS
            assert np.all(col >= 0)
        eng.update()
        delta1, b1, a1, s1, t1 = eng.read_state()
        del eng, k
    finally:
        _release()
    # the O(n) update applied by the oracle to the GPU's own columns
    delta, b, a0, s, t = st
    c_tilde = c + oprm.alpha / n
    d_bar = O._mirror(delta, col_now, c, c_tilde, oprm, 1.0)
    d_next = np.clip(O._mirror(delta, col_bar, c, c_tilde, oprm, 1.0), -oprm.beta, oprm.beta)
    ea, eb, es, et = O._advance(a0, b, s, t, np.tanh(0.5 * d_bar), oprm, 1.0)
    assert rel_err(delta1, d_next) <= TOL_UPDATE
    assert rel_err(b1, eb) <= TOL_UPDATE
    assert a1 == ea and abs(s1 - es) <= 1e-15 and t1 == et
    # sampled row blocks: the partial over those rows, all 1e5 columns, vs the oracle
    for i0 in (0, 49_968, n - 64):
        i1 = i0 + 64
        kb = core.HashKernel(n, seed=7, rows=(i0, i1))
        eb_ = _engine(kb, r, c, prm, st)
        part_now, part_bar = _cols(eb_)
        ref_now, ref_bar = _oracle_block(hc.block(i0, i1), r, ws, i0, i1)
        assert rel_err(part_now, ref_now) <= TOL_BLOCK, i0
        assert rel_err(part_bar, ref_bar) <= TOL_BLOCK, i0
        assert abs(part_now.sum() - r[i0:i1].sum()) <= TOL_MASS * r[i0:i1].sum() + 1e-17
        del eb_, kb


def test_config4_shard_full_width_properties():
    """BASELINE config 4: n = 1e6 3-D points on the fly, one 1/8 row shard (the per-GPU work)."""
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import shard_rows
    n = 1_000_000
    rng = np.random.default_rng(4)
    f = rng.random((n, 3))
    f[0], f[1] = 0.0, 1.0
    r, c = _hist(rng, n), _hist(rng, n)
    prm = dxg.params_tuned(1e-7).with_overrides(tau_mu=0.05)
    oprm = O.params_tuned(1e-7, tau_mu=0.05)
    st = _state(rng, n, 300.0)
    r0, r1 = shard_rows(n, 8, 7)
    k = core.ColorKernel(f, 2, scale=3.0)
    k.row0, k.row1 = r0, r1
    eng = _engine(k, r, c, prm, st)
    col_now, col_bar = _cols(eng)
    for col in (col_now, col_bar):
        assert abs(col.sum() - r[r0:r1].sum()) <= TOL_MASS
    del eng
    pc = O.PointCost(f, 2, scale=3.0)
    ws = [(st[2], st[1]), _bar_weights(st, oprm, 1.0)]
    for i0 in (r0, r1 - 16):
        i1 = i0 + 16
        kb = core.ColorKernel(f, 2, scale=3.0)
        kb.row0, kb.row1 = i0, i1
        e = _engine(kb, r, c, prm, st)
        part_now, part_bar = _cols(e)
        ref_now = np.zeros(n)
        ref_bar = np.zeros(n)
        for j0 in range(i0, i1, 4):
            pn, pb = _oracle_block(pc.block(j0, j0 + 4), r, ws, j0, j0 + 4)
            ref_now += pn
            ref_bar += pb
        assert rel_err(part_now, ref_now) <= TOL_BLOCK, i0
        assert rel_err(part_bar, ref_bar) <= TOL_BLOCK, i0
        del e, kb
    _release()


def test_shard_partials_sum_to_unsharded_columns():
    """Row shards summed in rank order (the multi-GPU combine) == one unsharded sweep, n = 1e5."""
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import shard_rows
    n = 100_000
    rng = np.random.default_rng(11)
    f = rng.random((n, 3))
    r, c = _hist(rng, n), _hist(rng, n)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    st = _state(rng, n, 400.0)
    full = _cols(_engine(core.ColorKernel(f, 2), r, c, prm, st))
    acc = [np.zeros(n), np.zeros(n)]
    for rank in range(4):
        k = core.ColorKernel(f, 2)
        k.row0, k.row1 = shard_rows(n, 4, rank)
        part = _cols(_engine(k, r, c, prm, st))
        acc[0] += part[0]
        acc[1] += part[1]
    assert rel_err(acc[0], full[0]) <= 1e-13
    assert rel_err(acc[1], full[1]) <= 1e-13
    _release()
