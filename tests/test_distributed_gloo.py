"""Row-sharded DXG across 2 processes over gloo (CPU): the host-side sharding and
column-partial combine used on multi-GPU runs (engine.shard_rows / combine_partials).

Each rank sweeps only its rows (oracle restatement as the per-rank compute, since
there is no GPU here); the combined column marginals must equal the unsharded
sweep, and a few full DXG iterations driven through the sharded combine must
track the unsharded iterate.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    import leanot_oracle as O
    from paper_2511_11359_b200.engine import combine_partials, shard_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, q, O, combine_partials, shard_rows)
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


def _body(rank, world, q, O, combine_partials, shard_rows):
    if True:
        rng = np.random.default_rng(11)
        n = 301
        Cm = rng.random((n, n))
        r = O.normalized_hist(rng.random(n))
        c = O.normalized_hist(rng.random(n))
        cost = O.DenseCost(Cm)
        prm = O.params_tuned(0.0, tau_mu=0.05)
        r0, r1 = shard_rows(n, world, rank)

        class Shard:
            def __init__(self):
                self.n, self.sup_norm = n, cost.sup_norm

            def block(self, i0, i1):
                return cost.block(i0, i1)

        def sharded_cols(it):
            a_bar, b_bar, _, _ = O._advance(it.a, it.b, it.s, it.t, np.tanh(0.5 * it.delta), prm, cost.sup_norm)
            rr = np.zeros(n)
            rr[r0:r1] = r[r0:r1]          # rows outside the shard carry no mass here
            parts = O.column_marginals(cost, rr, [(it.a, it.b), (a_bar, b_bar)])
            local = torch.from_numpy(np.concatenate(parts))
            return combine_partials(local, dist.group.WORLD, world).numpy()

        it_full = O.Iterate.zero(n)
        it_sh = O.Iterate.zero(n)
        errs = []
        for _ in range(5):
            cols = sharded_cols(it_sh)
            _, cn, cb = O.step(it_full, cost, r, c, prm, return_cols=True)
            errs.append(float(np.max(np.abs(cols - np.concatenate([cn, cb])))))
            it_full = O.step(it_full, cost, r, c, prm)
            # advance the sharded iterate with the combined marginals (same O(n) update)
            n_ = n
            c_tilde = c + prm.alpha / n_
            a_bar, b_bar, s_bar, t_bar = O._advance(it_sh.a, it_sh.b, it_sh.s, it_sh.t,
                                                    np.tanh(0.5 * it_sh.delta), prm, 1.0)
            d_bar = O._mirror(it_sh.delta, cols[:n], c, c_tilde, prm, 1.0)
            d_next = np.clip(O._mirror(it_sh.delta, cols[n:], c, c_tilde, prm, 1.0), -prm.beta, prm.beta)
            a, b, s, t = O._advance(it_sh.a, it_sh.b, it_sh.s, it_sh.t, np.tanh(0.5 * d_bar), prm, 1.0)
            it_sh = O.Iterate(d_next, a, b, s, t)
        scal = combine_partials(torch.tensor([float(rank + 1), 2.0 * rank]), dist.group.WORLD, world)
        q.put((rank, max(errs), float(np.max(np.abs(it_sh.delta - it_full.delta))), scal.tolist(), (r0, r1)))


@pytest.mark.parametrize("world", [2])
def test_row_sharded_iterations_match_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    for r in res:
        assert not isinstance(r[1], str), r[1]
    shards = [r[4] for r in res]
    assert shards[0][0] == 0 and shards[-1][1] == 301 and shards[0][1] == shards[1][0]
    for rank, col_err, delta_err, scal, _ in res:
        assert col_err <= 1e-16, col_err
        assert delta_err <= 1e-13, delta_err
        assert scal == [3.0, 2.0]


def test_shard_rows_cover_exactly():
    from paper_2511_11359_b200.engine import shard_rows
    for n in (1, 7, 100, 99856):
        for world in (1, 2, 3, 8):
            got = [shard_rows(n, world, k) for k in range(world)]
            covered = [i for a, b in got for i in range(a, b)]
            assert covered == list(range(n))
