"""Row-sharded solves through a REAL process group (needs a B200).

Two processes share the one GPU a gpurun box has and form a `gloo` group (device tensors
are staged through host memory by engine.all_gather_flat / all_reduce_max; on an 8 x B200
node the same code runs over NCCL).  No kernel waits on another process: each rank sweeps
its own rows and the collectives run on the host.  dxg.solve / dxgb_solve pick the group up
from torch.distributed (engine.default_group), shard the rows of the cost, and exchange the
2n column partials (barycenter: 2mn + the r-map normalizers) every iteration, summed in rank
order (core.py:297-309 / dxg.py:205-207 across ranks).

Grid costs (BASELINE config 5) run the separable O(n^1.5) path, which is not row-sharded:
every rank runs the whole iteration (replicas; no per-iteration collective), so the result
is bitwise the single-process one.

Checked against the single-process run of the same instance: identical iteration counts
and converged flags, trajectory and final state within 1e-10 (the sharded sum adds the same
terms in a different fixed order).
"""

import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dxg_instance(n=2048):
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(3)
    k = core.HashKernel(n, seed=3)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    return k, r, c, prm, dxg.Termination(eps=2e-3, max_iter=4000)


def _bary_instance(kind="points"):
    """points: a dense (row-sharded) barycenter; grid: the separable path (replicated per rank)."""
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(4)
    g = core.GridKernel(12, 12, 2) if kind == "grid" else core.ColorKernel(rng.random((150, 2)), 2)
    margs = [core.Histogram.normalized(rng.random(g.n) + 0.05) for _ in range(3)]
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    return g, margs, np.array([0.2, 0.5, 0.3]), prm, dxg.Termination(eps=5e-3, max_iter=3000)


def _run(which, timeout=None):
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import dxg
    if which == "dxg":
        k, r, c, prm, term = _dxg_instance()
        if timeout is not None:
            term = dxg.Termination(eps=1e-12, max_iter=10**6, timeout=timeout)
        sol = dxg.solve(k, r, c, prm, term, log_stride=25, dense_cap=0)
        traj = np.array([[p.iter, p.primal, p.dual, p.col_infeas_l1] for p in sol.trajectory])
        return dict(iterations=sol.iterations, converged=sol.converged, traj=traj, delta=sol.state.mu.delta,
                    b=sol.state.weights.b)
    g, margs, w, prm, term = _bary_instance("grid" if which == "bary_grid" else "points")
    sol = B.dxgb_solve(g, margs, w, prm, term, log_stride=25)
    traj = np.array([[p.iter, p.primal, p.dual, p.col_infeas_l1] for p in sol.trajectory])
    return dict(iterations=sol.iterations, converged=sol.converged, traj=traj, bary=sol.barycenter.weights,
                deltas=sol.state.deltas)


def _worker(rank, world, port, which, out, timeout):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(which, timeout)
        np.savez(f"{out}_{rank}.npz", **{k: np.asarray(v) for k, v in res.items()})
    finally:
        dist.destroy_process_group()


def _spawn(which, timeout=None):
    import torch.multiprocessing as mp
    d = tempfile.mkdtemp()
    out = os.path.join(d, which)
    mp.spawn(_worker, args=(2, _free_port(), which, out, timeout), nprocs=2, join=True)
    return [dict(np.load(f"{out}_{q}.npz")) for q in range(2)]


@pytest.mark.parametrize("which", ["dxg", "bary", "bary_grid"])
def test_two_rank_solve_matches_single_process(which):
    ranks = _spawn(which)
    single = _run(which)
    for res in ranks:
        assert int(res["iterations"]) == single["iterations"]
        assert bool(res["converged"]) == single["converged"]
        assert res["traj"].shape == single["traj"].shape
        assert np.array_equal(res["traj"][:, 0], single["traj"][:, 0])
        assert rel_err(res["traj"][:, 1:], single["traj"][:, 1:]) <= 1e-10
    for key in ("delta", "b") if which == "dxg" else ("bary", "deltas"):
        assert np.array_equal(ranks[0][key], ranks[1][key])         # identical on every rank
        assert rel_err(ranks[0][key], single[key]) <= 1e-10
        if which == "bary_grid":     # separable path replicated per rank: the same launches
            assert np.array_equal(ranks[0][key], single[key])


def test_two_rank_timeout_is_agreed():
    """A wall-clock timeout stops both ranks at the same iteration (engine.any_rank): without
    the agreement one rank would enter the evaluation collectives alone and hang."""
    ranks = _spawn("dxg", timeout=1.5)
    assert int(ranks[0]["iterations"]) == int(ranks[1]["iterations"])
    assert not bool(ranks[0]["converged"])
    assert np.array_equal(ranks[0]["traj"], ranks[1]["traj"][:, :]) or \
        np.array_equal(ranks[0]["traj"][:, 0], ranks[1]["traj"][:, 0])
