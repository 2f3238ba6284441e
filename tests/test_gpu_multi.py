"""Device side of the multi-GPU combine (needs a B200; the collective itself is covered by the
gloo tests in test_distributed_gloo.py -- a gpurun box has one GPU).

engine.combine_partials all-gathers the ranks' row-shard partials and sums them in rank
order with leanot_sum_partials, so the result is bitwise identical on every rank and equal
to a fixed-order host sum."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,count", [(1, 7), (2, 200_001), (8, 2 * 100_000), (3, 5)])
def test_sum_partials_rank_order_bitwise(world, count):
    import torch
    from paper_2511_11359_b200 import _lib
    rng = np.random.default_rng(world + count)
    g = rng.standard_normal((world, count)) * np.exp(rng.uniform(-30, 30, (world, count)))
    dev = torch.from_numpy(g.reshape(-1)).cuda()
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().leanot_sum_partials(dev.data_ptr(), world, count, out.data_ptr(), _lib.stream_handle()),
               "sum_partials")
    ref = g[0].copy()
    for q in range(1, world):
        ref += g[q]
    assert np.array_equal(out.cpu().numpy(), ref)


def test_engine_shards_combine_to_unsharded_sweep():
    """Two row shards swept on one GPU and combined with the device rank-order sum equal the
    unsharded sweep (the per-iteration exchange of the 2n column partials, engine.sweep)."""
    import torch
    from paper_2511_11359_b200 import _lib, core, dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n = 20000
    rng = np.random.default_rng(3)
    r = rng.random(n); r /= r.sum()
    c = rng.random(n); c /= c.sum()
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 20, n)); b -= b.max()
    cols = []
    for rows in ((0, 12345), (12345, n), None):
        k = core.HashKernel(n, seed=5, rows=rows) if rows else core.HashKernel(n, seed=5)
        eng = DxgEngine(k, r, c, prm)
        eng.load_state(delta, b, 400.0, 0.1, 50)
        eng.sweep()
        cols.append(eng.col.clone())
        del eng, k
    gathered = torch.cat([cols[0], cols[1]])
    out = torch.empty_like(cols[0])
    _lib.check(_lib.lib().leanot_sum_partials(gathered.data_ptr(), 2, cols[0].numel(), out.data_ptr(),
                                              _lib.stream_handle()), "sum_partials")
    full = cols[2].cpu().numpy()
    got = out.cpu().numpy()
    assert np.max(np.abs(got - full)) <= 1e-13 * np.max(np.abs(full))


def _bary_setup(n, m, seed):
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(seed)
    f = rng.random((n, 2))
    marg = [core.Histogram.normalized(rng.random(n)) for _ in range(m)]
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    return f, marg, prm


def _kernel_rows(f, rows):
    from paper_2511_11359_b200 import core
    k = core.ColorKernel(f, 2, scale=2.0)
    if rows is not None:
        k.row0, k.row1 = rows
    return k


def test_sharded_barycenter_matches_single_process():
    """Barycenter row sharding: two row shards driven in lockstep on one GPU,
    with the three exchanges of a multi-GPU iteration done here (max of the r-map maxima,
    rank-order sums of the exp-sums and of the 2 m n column partials), track the
    single-process barycenter iteration and evaluation."""
    import torch
    from paper_2511_11359_b200 import _lib
    from paper_2511_11359_b200.barycenter import BaryEngine, _combine_eval_buffers
    n, m, iters = 3000, 3, 6
    f, marg, prm = _bary_setup(n, m, 7)
    w = np.array([0.2, 0.5, 0.3])
    full = BaryEngine(_kernel_rows(f, None), marg, w, prm)
    shards = [BaryEngine(_kernel_rows(f, rows), marg, w, prm) for rows in ((0, 1401), (1401, n))]
    assert all(e.sharded for e in shards) and not full.sharded
    rng = np.random.default_rng(1)
    deltas = rng.uniform(-1, 1, (m, n))
    bs = -np.abs(rng.normal(0, 3, (m, n)))
    bs -= bs.max(axis=1, keepdims=True)
    for e in [full] + shards:
        e.load_state(deltas, bs, 20.0, 0.01, 40)

    def rank_sum(ts):
        g = torch.cat([t.reshape(-1) for t in ts])
        out = torch.empty_like(ts[0].reshape(-1))
        _lib.check(_lib.lib().leanot_sum_partials(g.data_ptr(), len(ts), out.numel(), out.data_ptr(),
                                                  _lib.stream_handle()), "sum_partials")
        return out.view(ts[0].shape)

    def sharded_sweep(evaluate=False):
        for e in shards:
            e.sweep_rows(evaluate)
        gm = torch.maximum(shards[0].gmax, shards[1].gmax)
        for e in shards:
            e.gmax.copy_(gm)
            e.sweep_rnorm()
        es = rank_sum([e.esum for e in shards])
        for e in shards:
            e.esum.copy_(es)
            e.sweep_cols()
        col = rank_sum([e.col for e in shards])
        for e in shards:
            e.col.copy_(col)

    for _ in range(iters):
        full.sweep()
        full.update()
        sharded_sweep()
        for e in shards:
            e.update()
    st_full = full.read_state()
    for e in shards:
        st = e.read_state()
        assert np.max(np.abs(st[0] - st_full[0])) <= 1e-11 * np.max(np.abs(st_full[0]))
        assert np.max(np.abs(st[1] - st_full[1])) <= 1e-11 * np.max(np.abs(st_full[1]))
        assert st[2:] == st_full[2:]
    # evaluation: combined per-shard buffers == single-process buffer
    full.sweep(evaluate=True)
    sharded_sweep(evaluate=True)
    r_full = full.r[:n].cpu().numpy()
    r_sh = np.concatenate([shards[0].r[:1401].cpu().numpy(), shards[1].r[1401:n].cpu().numpy()])
    assert np.max(np.abs(r_sh - r_full)) <= 1e-12 * np.max(r_full)
    full._call("leanot_bary_eval")
    bufs = []
    for e in shards:
        e._call("leanot_bary_eval")
        bufs.append(e.evalbuf.cpu().numpy())
    comb = _combine_eval_buffers(bufs, m)
    ref = full.evalbuf.cpu().numpy()
    for j in [4 * k for k in range(m)] + [4 * k + 1 for k in range(m)] + [64 + 2 * k for k in range(m)] + [127]:
        assert abs(comb[j] - ref[j]) <= 1e-11 * max(1.0, abs(ref[j])), j


def test_sharded_dxg_iterations_match_single_process():
    """DXG row sharding: two shards in lockstep on one GPU (the per-iteration exchange of the
    2n column partials done with the device rank-order sum), 10 iterations and an evaluation,
    against the unsharded engine."""
    import torch
    from paper_2511_11359_b200 import _lib, core, dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n, cut = 16000, 7001
    rng = np.random.default_rng(9)
    r = rng.random(n); r /= r.sum()
    c = rng.random(n); c /= c.sum()
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    engs = [DxgEngine(core.HashKernel(n, seed=2, rows=rows) if rows else core.HashKernel(n, seed=2), r, c, prm)
            for rows in (None, (0, cut), (cut, n))]
    for e in engs:
        e.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)

    def rank_sum(ts):
        g = torch.cat([t.reshape(-1) for t in ts])
        out = torch.empty_like(ts[0].reshape(-1))
        _lib.check(_lib.lib().leanot_sum_partials(g.data_ptr(), len(ts), out.numel(), out.data_ptr(),
                                                  _lib.stream_handle()), "sum_partials")
        return out

    full, s0, s1 = engs
    for it in range(10):
        ev = it == 9
        for e in engs:
            e.sweep(evaluate=ev)
        col = rank_sum([s0.col, s1.col])
        s0.col.copy_(col); s1.col.copy_(col)
        if ev:
            break
        for e in engs:
            e.update()
    assert np.max(np.abs(s0.col.cpu().numpy() - full.col.cpu().numpy())) <= 1e-13
    with torch.cuda.device(0):
        for e in engs:
            _lib.check(_lib.lib().leanot_dxg_eval(__import__("ctypes").byref(e.plan), _lib.stream_handle()), "eval")
    b_full = full.evalbuf[:5].cpu().numpy()
    rows = rank_sum([s0.evalbuf[:3], s1.evalbuf[:3]]).cpu().numpy()
    assert np.max(np.abs(rows - b_full[:3])) <= 1e-12 * np.max(np.abs(b_full[:3]))
    assert np.max(np.abs(s0.evalbuf[3:5].cpu().numpy() - b_full[3:5])) <= 1e-12 * np.max(np.abs(b_full[3:5]))
    d_full, b_f, a_f, s_f, t_f = full.read_state()
    d_0, b_0, a_0, s_0, t_0 = s0.read_state()
    assert np.max(np.abs(d_0 - d_full)) <= 1e-11 * max(1e-300, np.max(np.abs(d_full)))
    assert np.max(np.abs(b_0 - b_f)) <= 1e-11 * max(1.0, np.max(np.abs(b_f)))
    assert (a_0, s_0, t_0) == (a_f, s_f, t_f)


def test_sharded_points_expanded_form_matches_single_process():
    """Row shards of a squared-Euclidean point cost (expanded-form sweeps, global row norms and
    shifts per shard) combined in rank order equal the unsharded sweep and iteration."""
    import torch
    from paper_2511_11359_b200 import _lib, core, dxg
    from paper_2511_11359_b200.engine import DxgEngine
    n, cut = 9000, 4321
    rng = np.random.default_rng(21)
    f = rng.random((n, 3))
    r = rng.random(n); r /= r.sum()
    c = rng.random(n); c /= c.sum()
    prm = dxg.params_tuned(1e-4).with_overrides(tau_mu=0.05)

    def kern(rows):
        k = core.ColorKernel(f, 2, scale=3.0)
        if rows:
            k.row0, k.row1 = rows
        return k
    engs = [DxgEngine(kern(rows), r, c, prm) for rows in (None, (0, cut), (cut, n))]
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 30, n)); b -= b.max()
    for e in engs:
        e.load_state(delta, b, 300.0, 0.01, 30)
    full, s0, s1 = engs
    for _ in range(5):
        for e in engs:
            e.sweep()
        g = torch.cat([s0.col, s1.col])
        out = torch.empty_like(s0.col)
        _lib.check(_lib.lib().leanot_sum_partials(g.data_ptr(), 2, out.numel(), out.data_ptr(), _lib.stream_handle()),
                   "sum_partials")
        s0.col.copy_(out); s1.col.copy_(out)
        assert np.max(np.abs(out.cpu().numpy() - full.col.cpu().numpy())) <= 1e-13
        for e in engs:
            e.update()
    d_f, b_f, a_f, s_f, t_f = full.read_state()
    d_0, b_0, a_0, s_0, t_0 = s0.read_state()
    assert np.max(np.abs(d_0 - d_f)) <= 1e-11 and np.max(np.abs(b_0 - b_f)) <= 1e-11 * max(1.0, np.max(np.abs(b_f)))
