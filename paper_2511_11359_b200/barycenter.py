"""DXG for entropic OT barycenters on B200 -- drop-in for leanot.barycenter.

Same names, arguments and dataclasses as the reference
(/root/reference/pkg/src/leanot/barycenter.py).  One iteration is one device
sweep per marginal over both half-steps' weight sets, the sorted k-sum r-map and
one column pass per marginal (libleanot_b200.so: leanot_bary_*); evaluation is
folded into the next iteration's sweep like in dxg.solve.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CostKernel, Histogram, as_device_kernel, as_weights
from .engine import any_rank, default_group
from .dxg import (DxgParams, LogOddsField, Termination, TrajectoryPoint, TransportLogWeights, _plan_stats,
                  _to_dev, _ws, _wsets)

__all__ = ["BarycenterState", "BarycenterSolution", "barycenter_marginal", "dxgb_step", "dxgb_solve",
           "barycenter_objective"]


def _torch():
    import torch
    return torch


@dataclass
class BarycenterState:
    """barycenter.py:44-75."""

    deltas: np.ndarray
    bs: np.ndarray
    a: float
    s: float
    t: int
    w: np.ndarray
    eta: float

    @classmethod
    def initial(cls, n: int, weights, eta: float) -> "BarycenterState":
        if eta <= 0:
            raise ValueError("barycenter solver requires eta > 0")
        w = np.asarray(weights, dtype=float).ravel()
        if np.any(w <= 0):
            raise ValueError("weights must be positive")
        w = w / w.sum()
        m = w.size
        return cls(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, w, eta)

    @property
    def m(self) -> int:
        return self.w.size

    def weights_k(self, k: int) -> TransportLogWeights:
        return TransportLogWeights(self.a, self.bs[k], self.s, self.t)

    def mu_k(self, k: int) -> LogOddsField:
        return LogOddsField(self.deltas[k])


@dataclass
class BarycenterSolution:
    barycenter: Histogram
    state: BarycenterState
    converged: bool
    iterations: int
    seconds: float
    trajectory: list[TrajectoryPoint]
    per_marginal_infeas: np.ndarray = field(default=None)
    workers: int = 1

    @property
    def final(self) -> TrajectoryPoint:
        return self.trajectory[-1]


class BaryEngine:
    """Device state + workspaces of one barycenter solve.

    With a torch.distributed group (one process per GPU) the rows of the cost are
    sharded (engine.shard_rows); per iteration the ranks exchange the two r-map
    normalizers (max, then rank-order sum of the exp-sums) and the 2 m n column
    partials (rank-order sum); the O(n) updates run redundantly.
    """

    def __init__(self, kernel: CostKernel, marginals, w, params: DxgParams, group=None):
        torch = _torch()
        self.kernel = kernel
        self.device = dev = kernel.device
        n = self.n = kernel.n
        self.group, self.world, self.rank = group, 1, 0
        if group is not None:
            import torch.distributed as dist
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        r0, r1 = kernel.local_rows
        if self.world > 1 and kernel.cost_struct().kind == _lib.COST_GRID and (r0, r1) == (0, n):
            # grid costs run the separable O(n^1.5) sweeps (leanot_sep.cu; config 5: 0.54 ms per
            # iteration on one GPU).  Sharding their rows would put an exchange between every
            # LSE-convolution stage for no gain, so every rank runs the whole iteration
            # (identical on all ranks: replicas, no collective per iteration)
            self.world, self.rank = 1, 0
        if self.world > 1 and (r0, r1) == (0, n):
            from .engine import shard_rows
            r0, r1 = shard_rows(n, self.world, self.rank)
        self.row0, self.row1 = r0, r1
        self.sharded = (r0, r1) != (0, n)
        M = np.stack([as_weights(h) for h in marginals])
        m = self.m = M.shape[0]
        if M.shape[1] != n:
            raise ValueError("state/marginal/kernel size mismatch")
        wv = np.asarray(w, dtype=float).ravel()
        self.params = params
        L = _lib.lib()
        s = C.c_int(1)
        L.leanot_dxg_default_splits(n, n, C.byref(s))
        splits = s.value
        sms = C.c_int(148)
        L.leanot_device_sm_count(dev.index or 0, C.byref(sms))
        nblk = int(min(max(1, (n + 255) // 256), 2 * sms.value))
        f64 = dict(dtype=torch.float64, device=dev)
        ns = self.ns = n + (-n) % 4                      # 16-byte aligned per-marginal slices
        self.w = torch.from_numpy(wv).to(dev)
        z = lambda *shape: torch.zeros(*shape, **f64)   # noqa: E731
        self.c = z(m, ns)
        self.c[:, :n] = torch.from_numpy(np.ascontiguousarray(M)).to(dev)
        self.c_tilde = self.c + params.alpha / n          # c_k + alpha/n (barycenter.py:130)
        self.delta, self.b, self.b_bar, self.bprime, self.sd = (z(m * ns) for _ in range(5))
        self.scal = z(8)
        self.shift = torch.zeros(m * n, dtype=torch.int64, device=dev)
        self.mu = torch.zeros(2 * m * n, dtype=torch.int64, device=dev)
        self.S = z(2 * m * n)
        self.L = z(2 * m * n)
        self.r = z(2 * n)
        self.coef = z(8 * m * n)
        self.rowstat = z(3 * m * n)
        slab = splits * 4 * n     # pass B of two marginals at once (K = 4 weight sets, leanot_bary.cu)
        if kernel.cost_struct().kind == _lib.COST_GRID:   # separable path scratch (leanot_sep.cu)
            cs = kernel.cost_struct()
            slab = max(slab, int(L.leanot_grid_sep_ws_doubles(cs)) + 5 * m * n + m * max(cs.height, cs.width))
        self.slab = z(slab)
        self.col = z(2 * m * n)
        self.partial = z(2 * m * max(nblk, (n + 255) // 256) + 2048)   # batched update: 2 nblk per marginal
        self.scratch = z(n)
        self.evalbuf = z(128)
        self.flags = torch.zeros(2 + 4 * n, dtype=torch.int32, device=dev)
        p = self.plan = _lib.BaryPlanT()
        p.cost = kernel.cost_struct()
        p.prm = _lib.ParamsT(params.eta, params.eta_mu, params.tau_p, params.tau_mu, params.beta, params.alpha)
        p.n, p.row0, p.row1, p.ns, p.m, p.splits, p.nblk_upd = n, r0, r1, ns, m, int(splits), nblk
        self.gmax = z(2)   # sharded sweeps: r-map normalizers (leanot_bary_rows / _rnorm)
        self.esum = z(2)
        for name in ("w", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "mu", "S", "L",
                     "r", "coef", "rowstat", "slab", "col", "partial", "scratch", "evalbuf", "flags"):
            setattr(p, name, getattr(self, name).data_ptr())
        self.M = M
        self.wv = wv
        self._h_in = self._h_out = None

    def _call(self, name, *args):
        with _torch().cuda.device(self.device):
            _lib.check(getattr(_lib.lib(), name)(C.byref(self.plan), *args, _lib.stream_handle()), name)

    def _staging(self):
        """Pinned host buffers (deltas | bs, and + 4 scalars on the way out) and their device
        mirror: one async H2D per load, one synchronisation per read."""
        torch = _torch()
        if self._h_in is None:
            k = 2 * self.m * self.n
            self._h_in = torch.empty(k, dtype=torch.float64, pin_memory=True)
            self._h_out = torch.empty(k + 4, dtype=torch.float64, pin_memory=True)
            self._d_stage = torch.empty(k + 4, dtype=torch.float64, device=self.device)
            self._h_in_done = torch.cuda.Event()
        return self._h_in, self._h_out, self._d_stage

    def load_state(self, deltas, bs, a, s, t, fresh=False):
        torch = _torch()
        m, n, ns = self.m, self.n, self.ns
        first = self._h_in is None
        h_in, _, d = self._staging()
        if not first:
            self._h_in_done.synchronize()   # the previous upload has left the staging buffer
        hv = h_in.numpy().reshape(2, m, n)
        hv[0] = np.asarray(deltas, dtype=float).reshape(m, n)
        hv[1] = np.asarray(bs, dtype=float).reshape(m, n)
        with torch.cuda.device(self.device):
            d[: 2 * m * n].copy_(h_in, non_blocking=True)
            self._h_in_done.record()
            dv = d[: 2 * m * n].view(2, m, n)
            self.delta.view(m, ns)[:, :n].copy_(dv[0])
            self.b.view(m, ns)[:, :n].copy_(dv[1])
        self._call("leanot_bary_prepare", float(a), float(s), float(t), 1 if fresh else 0)

    def sweep(self, evaluate=False):
        if not self.sharded:
            self._call("leanot_bary_sweep", 1 if evaluate else 0)
            return
        from .engine import all_reduce_max, combine_partials
        self.sweep_rows(evaluate)
        if self.world > 1:
            self.gmax.copy_(all_reduce_max(self.gmax, self.group))   # order-independent
        self.sweep_rnorm()
        if self.world > 1:
            self.esum.copy_(combine_partials(self.esum, self.group, self.world))
        self.sweep_cols()
        if self.world > 1:
            self.col.copy_(combine_partials(self.col, self.group, self.world))

    # the three phases of a row-sharded sweep (leanot_bary_rows / _rnorm / _cols); sweep()
    # puts the collectives between them
    def sweep_rows(self, evaluate=False):
        self._call("leanot_bary_rows", 1 if evaluate else 0, self.gmax.data_ptr())

    def sweep_rnorm(self):
        self._call("leanot_bary_rnorm", self.gmax.data_ptr(), self.esum.data_ptr())

    def sweep_cols(self):
        self._call("leanot_bary_cols", self.esum.data_ptr())

    def update(self):
        self._call("leanot_bary_update")

    def read_state(self):
        torch = _torch()
        m, n, ns = self.m, self.n, self.ns
        _, h_out, d = self._staging()
        k = 2 * m * n
        with torch.cuda.device(self.device):
            dv = d[:k].view(2, m, n)
            dv[0].copy_(self.delta.view(m, ns)[:, :n])
            dv[1].copy_(self.b.view(m, ns)[:, :n])
            d[k:].copy_(self.scal[:4])
            h_out.copy_(d, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        ho = h_out.numpy()
        sc = ho[k:].tolist()
        return ho[: m * n].reshape(m, n).copy(), ho[m * n: k].reshape(m, n).copy(), sc[0], sc[2], int(round(sc[3]))

    def barycenter(self):
        """r_now of the last sweep = barycenter_marginal(state) (barycenter.py:100-105)."""
        if self.world > 1:
            return self._gather_rows(self.r[: self.n]).cpu().numpy()
        return self.r[: self.n].cpu().numpy()

    def _combine_eval(self):
        torch = _torch()
        import torch.distributed as dist
        from .engine import all_gather_flat
        gathered = all_gather_flat(self.evalbuf, self.group, self.world)
        bufs = gathered.view(self.world, -1).cpu().numpy()
        self.evalbuf.copy_(torch.from_numpy(_combine_eval_buffers(bufs, self.m)))

    def _gather_rows(self, full):
        """Every rank's own rows of a length-n device vector, assembled on all ranks."""
        torch = _torch()
        import torch.distributed as dist
        from .engine import shard_rows
        per = (self.n + self.world - 1) // self.world
        buf = torch.zeros(per, dtype=full.dtype, device=full.device)
        buf[: self.row1 - self.row0] = full[self.row0:self.row1]
        from .engine import all_gather_flat
        out = all_gather_flat(buf, self.group, self.world)
        res = torch.empty_like(full)
        for q in range(self.world):
            a, b = shard_rows(self.n, self.world, q)
            res[a:b] = out[q * per: q * per + (b - a)]
        return res

    def evaluate(self):
        """(primal, dual, infeas[m]) of the state swept by the last sweep(evaluate=True)."""
        self._call("leanot_bary_eval")
        if self.world > 1:
            self._combine_eval()
        buf = self.evalbuf.cpu().numpy()
        eta, sup = self.params.eta, self.kernel.sup_norm
        r = self.barycenter()
        pos = r > 0
        h_r = float(-(r[pos] * np.log(r[pos])).sum())
        primal = 0.0
        infeas = np.empty(self.m)
        lead = 0.0
        for k in range(self.m):
            cost_k, ent_rows_k = buf[4 * k], buf[4 * k + 1]
            infeas[k], cd_k = buf[64 + 2 * k], buf[64 + 2 * k + 1]
            ent_k = ent_rows_k + h_r
            primal += self.wv[k] * (cost_k + 2.0 * sup * infeas[k] - eta * ent_k)   # barycenter.py:222
            lead += self.wv[k] * (-2.0 * sup * cd_k)                                # barycenter.py:192
        dual = lead - eta * float(buf[127])                                         # barycenter.py:195
        return primal, dual, infeas


def _combine_eval_buffers(bufs, m):
    """Rank-order combination of per-rank evaluation buffers (sharded plans): row sums
    [4k], [4k+1] add; column stats [64+2k], [65+2k] are identical on every rank; [127] is a
    log-sum-exp over each rank's rows: M + log(sum_q exp(l_q - M)), q in rank order."""
    out = np.array(bufs[0], dtype=float)
    for k in range(m):
        for j in (4 * k, 4 * k + 1):
            v = bufs[0][j]
            for q in range(1, len(bufs)):
                v += bufs[q][j]
            out[j] = v
    ls = [float(b[127]) for b in bufs]
    M = max(ls)
    tot = 0.0
    for v in ls:
        tot += float(np.exp(v - M))
    out[127] = M + float(np.log(tot))
    return out


def _log_normalizers(a: float, bs: np.ndarray, kernel: CostKernel, workers: int = 1) -> np.ndarray:
    """(m, n) LSE_j(-(a C_ij + b_kj)) (barycenter.py:78-87), one device sweep per marginal."""
    torch = _torch()
    dev = kernel.device
    m, n = bs.shape
    with torch.cuda.device(dev):
        bt = [_to_dev(bs[k], dev) for k in range(m)]
        w, keep = _wsets(dev, [(a, b) for b in bt])
        out = torch.empty(m * n, dtype=torch.float64, device=dev)
        ws = _ws(kernel, 1, n)
        _lib.check(_lib.lib().leanot_row_lse(kernel.cost_struct(), 0, n, C.byref(w), out.data_ptr(), ws.data_ptr(),
                                             _lib.stream_handle()), "row_lse")
        res = out.view(m, n).cpu().numpy()
        del keep
    return res


def _marginal_from_logz(w: np.ndarray, log_z: np.ndarray, device) -> Histogram:
    """Sorted k-sum r-map on device (barycenter.py:90-97)."""
    torch = _torch()
    m, n = log_z.shape
    with torch.cuda.device(device):
        Lt = _to_dev(np.ascontiguousarray(log_z), device)
        wt = _to_dev(w, device)
        r = torch.empty(n, dtype=torch.float64, device=device)
        scratch = torch.empty(n + 4096, dtype=torch.float64, device=device)
        _lib.check(_lib.lib().leanot_bary_rmap(Lt.data_ptr(), m, n, wt.data_ptr(), r.data_ptr(), scratch.data_ptr(),
                                               _lib.stream_handle()), "bary_rmap")
        return Histogram(r.cpu().numpy())


def barycenter_marginal(state: BarycenterState, kernel: CostKernel, workers: int = 1) -> Histogram:
    """r_i proportional to exp(sum_k w_k log Z_ki) (barycenter.py:100-105)."""
    if state.eta <= 0:
        raise ValueError("barycenter map requires eta > 0")
    kernel = as_device_kernel(kernel)
    return _marginal_from_logz(state.w, _log_normalizers(state.a, state.bs, kernel, workers), kernel.device)


def dxgb_step(state: BarycenterState, kernel: CostKernel, marginals, params: DxgParams,
              workers: int = 1) -> BarycenterState:
    """One extragradient iteration across all marginals (barycenter.py:108-151)."""
    if params.eta <= 0:
        raise ValueError("barycenter solver requires eta > 0")
    m, n = state.deltas.shape
    if len(marginals) != m or kernel.n != n:
        raise ValueError("state/marginal/kernel size mismatch")
    kernel = as_device_kernel(kernel)
    eng = BaryEngine(kernel, marginals, state.w, params, group=default_group())
    eng.load_state(state.deltas, state.bs, state.a, state.s, state.t, fresh=False)
    eng.sweep()
    eng.update()
    deltas, bs, a, s, _ = eng.read_state()
    return BarycenterState(deltas, bs, a, s, state.t + 1, state.w, state.eta)


def barycenter_objective(state: BarycenterState, kernel: CostKernel, marginals, w=None, eta: float | None = None,
                         workers: int = 1) -> float:
    """sum_k w_k (<C, D_r p_k> + 2||C|| ||c(D_r p_k) - c_k||_1 - eta H(D_r p_k)) (barycenter.py:154-169)."""
    weights = state.w if w is None else np.asarray(w, dtype=float) / np.sum(w)
    eta_val = state.eta if eta is None else eta
    kernel = as_device_kernel(kernel)
    r = barycenter_marginal(state, kernel, workers)
    total = 0.0
    for k in range(len(marginals)):
        cost, col, ent = _plan_stats(state.weights_k(k), kernel, r, workers)
        pen = 2.0 * kernel.sup_norm * float(np.abs(col - as_weights(marginals[k])).sum())
        total += weights[k] * (cost + pen - eta_val * ent)
    return total


def dxgb_solve(kernel: CostKernel, marginals, w, params: DxgParams, termination: Termination = Termination(),
               log_stride: int = 25, workers: int = 1) -> BarycenterSolution:
    """Iterate to gap and worst column infeasibility <= eps/6 (barycenter.py:227-277)."""
    if params.eta <= 0:
        raise ValueError("barycenter solver requires eta > 0")
    kernel = as_device_kernel(kernel)
    torch = _torch()
    state0 = BarycenterState.initial(kernel.n, w, params.eta)
    eng = BaryEngine(kernel, marginals, state0.w, params, group=default_group())
    eng.load_state(state0.deltas, state0.bs, 0.0, 0.0, 0, fresh=True)
    t0 = time.perf_counter()
    trajectory: list[TrajectoryPoint] = []
    converged = False
    it = 0
    swept = False
    infeas = None

    def log_point():
        nonlocal swept, infeas
        if not swept:
            eng.sweep(evaluate=True)
            swept = True
        primal, dual, infeas = eng.evaluate()
        s_val = float(eng.scal[2].item())
        point = TrajectoryPoint(it, time.perf_counter() - t0, primal, dual, primal - dual, float(infeas.max()), s_val)
        trajectory.append(point)
        return point

    while it < termination.max_iter:
        if not swept:
            eng.sweep()
        eng.update()
        swept = False
        it += 1
        timed_out = False
        if termination.timeout is not None:
            torch.cuda.synchronize(eng.device)
            timed_out = time.perf_counter() - t0 > termination.timeout
            if eng.group is not None:   # every rank must take the same branch (collectives below)
                timed_out = any_rank(timed_out, eng.group)
        if it % log_stride == 0 or it == termination.max_iter or timed_out:
            eng.sweep(evaluate=True)
            swept = True
            point = log_point()
            if point.gap <= termination.eps / 6.0 and point.col_infeas_l1 <= termination.eps / 6.0:
                converged = True
                break
        if timed_out:
            break
    if not trajectory or trajectory[-1].iter != it:
        log_point()
    deltas, bs, a, s, _ = eng.read_state()
    state = BarycenterState(deltas, bs, a, s, it, state0.w, params.eta)
    return BarycenterSolution(barycenter=Histogram(eng.barycenter()), state=state, converged=converged,
                              iterations=it, seconds=time.perf_counter() - t0, trajectory=trajectory,
                              per_marginal_infeas=infeas, workers=workers)
