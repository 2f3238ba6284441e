"""Separable GridKernel path (O(n^1.5)) vs the dense n^2 sweeps and the oracle."""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


def _sep_col(kernel, a, b, r):
    import ctypes as C
    import torch
    from paper_2511_11359_b200 import _lib
    dev = kernel.device
    n = kernel.n
    L = _lib.lib()
    cs = kernel.cost_struct()
    ws = torch.empty(int(L.leanot_grid_sep_ws_doubles(cs)), dtype=torch.float64, device=dev)
    at = torch.tensor([a], dtype=torch.float64, device=dev)
    bt = torch.as_tensor(b, device=dev)
    Lr = torch.empty(n, dtype=torch.float64, device=dev)
    s = _lib.stream_handle()
    _lib.check(L.leanot_grid_sep_lse(cs, at.data_ptr(), bt.data_ptr(), Lr.data_ptr(), ws.data_ptr(), s))
    rt = torch.as_tensor(r, device=dev)
    logw = torch.where(rt > 0, torch.log(rt), torch.full_like(rt, -np.inf)) - Lr
    col = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(L.leanot_grid_sep_colsum(cs, at.data_ptr(), bt.data_ptr(), logw.data_ptr(), col.data_ptr(),
                                        ws.data_ptr(), s))
    return Lr.cpu().numpy(), col.cpu().numpy()


@pytest.mark.parametrize("H,W,p", [(8, 8, 1), (23, 17, 2), (40, 37, 3), (1, 30, 2), (64, 64, 2)])
def test_separable_matches_dense(H, W, p):
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(H * 100 + W)
    g = core.GridKernel(H, W, p)
    n = g.n
    r = O.normalized_hist(rng.random(n))
    r[rng.choice(n, max(1, n // 10), replace=False)] = 0.0
    r = r / r.sum()
    for a, bs in ((0.0, 0.0), (7.5, 2.0), (300.0, 40.0), (3000.0, 500.0)):
        b = -np.abs(rng.normal(0, bs, n)) if bs else np.zeros(n)
        Lsep, csep = _sep_col(g, a, b, r)
        cden = dxg.column_marginal(dxg.TransportLogWeights(a, b, 0, 0), g, r)
        (cor,) = O.column_marginals(O.GridCost(H, W, p), r, [(a, b)])
        assert rel_err(csep, cor) <= 1e-12, (a, bs)
        assert rel_err(cden, cor) <= 1e-12
        z = -(a * O.GridCost(H, W, p).block(0, n) + b[None, :])
        assert rel_err(Lsep, O.lse_rows(z)) <= 1e-13


def test_separable_solve_matches_reference_grid_run():
    """The golden grid solve (6x6, loose) goes through the separable sweep + separable evaluation."""
    from helpers import load
    from paper_2511_11359_b200 import core, dxg
    d = load("solve_grid_6x6_p2_loose")
    g = core.GridKernel(int(d["k_H"]), int(d["k_W"]), int(d["k_p"]))
    prm = dxg.DxgParams(*[float(v) for v in d["params"]])
    sol = dxg.solve(g, d["r"], d["c"], prm, dxg.Termination(eps=float(d["term"][0]), max_iter=int(d["term"][1])),
                    dense_cap=0)
    assert sol.iterations == int(d["iterations"]) and sol.converged == bool(d["converged"])
    got = np.array([[p.primal, p.dual] for p in sol.trajectory])
    assert rel_err(got, d["traj"][:, 1:3]) <= 1e-8


def test_separable_dxg_iterations_track_oracle_eta0():
    """Tuned + tau_mu=0.05 on a 30x30 grid (eta = 0 dual min-plus path), 60 iterations vs the oracle."""
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import DxgEngine
    rng = np.random.default_rng(9)
    H = W = 30
    n = H * W
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    eng = DxgEngine(core.GridKernel(H, W, 2), r, c, prm)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    og = O.GridCost(H, W, 2)
    it = O.Iterate.zero(n)
    oprm = O.params_tuned(0.0, tau_mu=0.05)
    for k in range(60):
        eng.sweep()
        eng.update()
        it = O.step(it, og, r, c, oprm)
    delta, b, a, s, t = eng.read_state()
    assert rel_err(delta, it.delta) <= 1e-10 and rel_err(b, it.b) <= 1e-10
    eng.sweep(evaluate=True)
    primal, dual, infeas = eng.evaluate()
    p2, d2, i2, _ = O.evaluate(it, og, r, c, 0.0)
    assert abs(primal - p2) <= 1e-11 and abs(dual - d2) <= 1e-11 and abs(infeas - i2) <= 1e-12


@pytest.mark.parametrize("a", [400.0, 2000.0])
def test_config5_grid_tensor_core_path_matches_dense(a):
    """316x316 grid (config 5 size): the separable sweep -- DMMA linear-domain GEMMs at a = 400,
    exact log-domain convolutions at a = 2000 (a * max f/scale > 600) -- against the dense n^2
    sweep of the same state (two row shards force the dense kernels, summed in rank order)."""
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import DxgEngine, shard_rows
    rng = np.random.default_rng(int(a))
    g = core.GridKernel(316, 316, 2)
    n = g.n
    r, c = O.normalized_hist(rng.random(n)), O.normalized_hist(rng.random(n))
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    delta = rng.uniform(-1, 1, n)
    b = -np.abs(rng.normal(0, 0.05 * a, n))
    b -= b.max()
    st = (delta, b, a, 0.2, 50)

    def cols(kernel):
        eng = DxgEngine(kernel, r, c, prm)
        eng.load_state(*st)
        eng.sweep()
        col = eng.col.cpu().numpy()
        return col[:n].copy(), col[n:].copy()

    sep = cols(g)
    dense = [np.zeros(n), np.zeros(n)]
    for rank in range(2):
        k = core.GridKernel(316, 316, 2)
        k.row0, k.row1 = shard_rows(n, 2, rank)
        part = cols(k)
        dense[0] += part[0]
        dense[1] += part[1]
    assert rel_err(sep[0], dense[0]) <= 1e-12
    assert rel_err(sep[1], dense[1]) <= 1e-12
