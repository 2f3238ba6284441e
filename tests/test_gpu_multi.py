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
