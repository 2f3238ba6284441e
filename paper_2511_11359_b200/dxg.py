"""Dual extragradient OT solver on B200 -- drop-in for leanot.dxg.

Same public names, arguments, dataclasses and error behaviour as the
reference (/root/reference/pkg/src/leanot/dxg.py); the n^2 sweeps and the
O(n) updates run in hand-written sm_100a kernels (csrc/), with the state in
HBM between iterations.  `workers` is accepted and recorded (the reference
threads over 128-row blocks) but the GPU ignores it.

Evaluation (dxg.py:412-417) is folded into the sweep of the next iteration:
the column marginal of _plan_stats is exactly the next iteration's col_now,
and <C, D_r p>, H(D_r p) and the eta = 0 dual row minima are extra per-row
accumulators of that same pass, so an evaluation costs no extra read of C.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .core import DENSE_CAP, CostKernel, Histogram, as_device_kernel, as_weights
from .engine import DxgEngine, any_rank, default_group
from .rounding import DenseCoupling, InfeasibilityReport, infeasibility, round_on_device, round_to_polytope
from .sinkhorn import DualPotentials

__all__ = [
    "LogOddsField", "TransportLogWeights", "DxgParams", "DxgState", "Termination", "TrajectoryPoint",
    "DxgSolution", "params_tuned", "params_li", "params_loose", "implicit_row", "column_marginal",
    "materialize_plan", "dual_md_step", "balance", "dxg_step", "primal_penalized_value",
    "dual_penalized_value", "recover_eot_potentials", "solve", "PdxgState", "pdxg_init",
    "pdxg_reference_step",
]


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class LogOddsField:
    """mu as per-column log-odds delta (dxg.py:57-79)."""

    delta: np.ndarray

    def diff(self) -> np.ndarray:
        return np.tanh(0.5 * self.delta)

    def mu_plus(self) -> np.ndarray:
        return 0.5 * (1.0 + self.diff())

    def mu_minus(self) -> np.ndarray:
        return 0.5 * (1.0 - self.diff())

    @classmethod
    def uniform(cls, n: int) -> "LogOddsField":
        return cls(np.zeros(n))


@dataclass(frozen=True)
class TransportLogWeights:
    """Implicit plan rows softmax(-(a C_i + b)) (dxg.py:82-97)."""

    a: float
    b: np.ndarray
    s: float
    t: int

    @classmethod
    def initial(cls, n: int) -> "TransportLogWeights":
        return cls(a=0.0, b=np.zeros(n), s=0.0, t=0)


@dataclass(frozen=True)
class DxgParams:
    """Stepsizes and regularization (dxg.py:100-128)."""

    eta: float
    eta_mu: float
    tau_p: float
    tau_mu: float
    beta: float
    alpha: float

    def __post_init__(self):
        if self.eta < 0 or self.eta_mu < 0:
            raise ValueError("eta and eta_mu must be nonnegative")
        if self.tau_p <= 0 or self.tau_mu <= 0:
            raise ValueError("stepsizes must be positive")
        if self.tau_p * self.eta >= 1 or self.tau_mu * self.eta_mu >= 1:
            raise ValueError("need tau_p*eta < 1 and tau_mu*eta_mu < 1")
        if self.beta <= 0:
            raise ValueError("beta must be positive")
        if not (0 <= self.alpha <= 1):
            raise ValueError("alpha must lie in [0, 1]")

    def with_overrides(self, **kw) -> "DxgParams":
        return replace(self, **kw)


def params_tuned(eta: float = 0.0) -> DxgParams:
    """dxg.py:131-133."""
    return DxgParams(eta=eta, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.01)


def params_li(n: int, eps: float, C1: float = 100.0, C2: float = 1.0, C3: float = 1.0) -> DxgParams:
    """dxg.py:136-154."""
    if n < 2 or eps <= 0:
        raise ValueError("need n >= 2 and eps > 0")
    if n / eps <= 1:
        raise ValueError("n/eps must exceed 1 (beta would be nonpositive)")
    if C1 <= 0 or C2 <= 0 or not (0 < C3 <= 1):
        raise ValueError("need C1 > 0, C2 > 0 and 0 < C3 <= 1")
    beta = C1 * math.log(n / eps)
    eta = eps * C2 * C2 / (math.sqrt(beta) * math.log(n))
    return DxgParams(eta=eta, eta_mu=eta, tau_p=C2 / math.sqrt(beta), tau_mu=15.0 * C2 * math.sqrt(beta),
                     beta=beta, alpha=C3)


def params_loose(n: int, eps: float, min_marginal: float, cost_sup: float = 1.0) -> DxgParams:
    """dxg.py:157-172."""
    if n < 2 or eps <= 0 or min_marginal <= 0 or cost_sup <= 0:
        raise ValueError("inputs must be positive (and n >= 2)")
    eta = min(cost_sup / (-math.log(min_marginal)), eps / (16.0 * math.log(n)))
    tau_mu = 1.0 / (4.0 * math.sqrt(n))
    min_ct = min_marginal + 1.0 / n
    tau_p = min_ct / (n ** -0.5 + eta * min_ct)
    eta_mu = min(eps / (16.0 * math.log(2.0)), eta * tau_p / tau_mu)
    return DxgParams(eta=eta, eta_mu=eta_mu, tau_p=tau_p, tau_mu=tau_mu, beta=math.log(3.0), alpha=1.0)


@dataclass(frozen=True)
class DxgState:
    mu: LogOddsField
    weights: TransportLogWeights

    @classmethod
    def initial(cls, n: int) -> "DxgState":
        return cls(LogOddsField.uniform(n), TransportLogWeights.initial(n))


@dataclass(frozen=True)
class Termination:
    """dxg.py:375-381."""

    eps: float = 1e-10
    max_iter: int = 1_000_000
    timeout: float | None = None


@dataclass(frozen=True)
class TrajectoryPoint:
    iter: int
    seconds: float
    primal: float
    dual: float
    gap: float
    col_infeas_l1: float
    s: float


@dataclass
class DxgSolution:
    state: DxgState
    converged: bool
    iterations: int
    seconds: float
    trajectory: list[TrajectoryPoint]
    report: InfeasibilityReport
    rounded_plan: DenseCoupling | None = None
    rounded_cost: float | None = None
    workers: int = 1

    @property
    def final(self) -> TrajectoryPoint:
        return self.trajectory[-1]


# ---------------------------------------------------------------------------
# sweeps through the C ABI
# ---------------------------------------------------------------------------


def _dev_kernel(kernel) -> CostKernel:
    return as_device_kernel(kernel)


def _wsets(dev, pairs):
    """Build a leanot_wsets_t from [(a, b_tensor)] with device scalars."""
    torch = _torch()
    a = torch.tensor([float(p[0]) for p in pairs], dtype=torch.float64, device=dev)
    w = _lib.WsetsT()
    w.K = len(pairs)
    w.a = a.data_ptr()
    for k, (_, b) in enumerate(pairs):
        w.b[k] = b.data_ptr()
    return w, a


def _ws(kernel, K, nr):
    torch = _torch()
    size = _lib.lib().leanot_sweep_ws_doubles(kernel.n, nr, K)
    return torch.empty(int(size), dtype=torch.float64, device=kernel.device)


def _to_dev(x, dev):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=float)), device=dev)


def _column_marginals(kernel: CostKernel, r_w, pairs):
    torch = _torch()
    dev = kernel.device
    r0, r1 = kernel.local_rows
    with torch.cuda.device(dev):
        bt = [_to_dev(b, dev) for _, b in pairs]
        w, keep = _wsets(dev, [(a, b) for (a, _), b in zip(pairs, bt)])
        rt = _to_dev(r_w, dev)
        out = torch.empty(len(pairs) * kernel.n, dtype=torch.float64, device=dev)
        ws = _ws(kernel, len(pairs), r1 - r0)
        _lib.check(_lib.lib().leanot_column_marginals(kernel.cost_struct(), r0, r1, C.byref(w), rt.data_ptr(),
                                                      out.data_ptr(), ws.data_ptr(), _lib.stream_handle()),
                   "column_marginals")
        res = out.view(len(pairs), kernel.n).cpu().numpy()
        del keep
    return res


def implicit_row(state: TransportLogWeights, kernel: CostKernel, i: int) -> np.ndarray:
    """Row i of the implicit plan (dxg.py:185-190), from a device cost row."""
    kernel = _dev_kernel(kernel)
    z = -(state.a * kernel.block(i, i + 1)[0] + np.asarray(state.b, dtype=float))
    e = np.exp(z - z.max())
    return e / e.sum()


def column_marginal(state: TransportLogWeights, kernel: CostKernel, r: Histogram, workers: int = 1) -> np.ndarray:
    """c(D_r p) in one device sweep (dxg.py:193-208)."""
    kernel = _dev_kernel(kernel)
    return _column_marginals(kernel, as_weights(r), [(state.a, state.b)])[0]


def _holds_all_rows(kernel) -> bool:
    return tuple(kernel.local_rows) == (0, kernel.n)


def _plan_on_device(state: TransportLogWeights, kernel: CostKernel, r_w):
    """D_r p as a device n x n tensor: row LSEs (sweep kernels) + one plan kernel."""
    torch = _torch()
    dev = kernel.device
    n = kernel.n
    if not _holds_all_rows(kernel):
        # a row-restricted stored cost (HashKernel(rows=...), one rank's shard) holds rows
        # [r0, r1) only: the dense plan would read rows it does not have
        r0, r1 = kernel.local_rows
        raise ValueError(f"the dense plan needs all {n} rows of the cost; this kernel holds rows [{r0}, {r1})")
    with torch.cuda.device(dev):
        bt = _to_dev(state.b, dev)
        w, keep = _wsets(dev, [(state.a, bt)])
        L = torch.empty(n, dtype=torch.float64, device=dev)
        ws = _ws(kernel, 1, n)
        lib = _lib.lib()
        s = _lib.stream_handle()
        _lib.check(lib.leanot_row_lse(kernel.cost_struct(), 0, n, C.byref(w), L.data_ptr(), ws.data_ptr(), s),
                   "row_lse")
        P = torch.empty((n, n), dtype=torch.float64, device=dev)
        rt = _to_dev(r_w, dev)
        _lib.check(lib.leanot_materialize_plan(kernel.cost_struct(), float(state.a), bt.data_ptr(), rt.data_ptr(),
                                               L.data_ptr(), P.data_ptr(), n, s), "materialize_plan")
        del keep
    return P


def materialize_plan(state: TransportLogWeights, kernel: CostKernel, r: Histogram, cap: int = DENSE_CAP) -> np.ndarray:
    """Dense D_r p for rounding and tests (dxg.py:211-220), computed on device."""
    kernel = _dev_kernel(kernel)
    if kernel.n > cap:
        raise ValueError("implicit plan materialization above the dense cap")
    return _plan_on_device(state, kernel, as_weights(r)).cpu().numpy()


def dual_md_step(mu: LogOddsField, col_marginal, c: Histogram, c_tilde, params: DxgParams,
                 sup_norm: float = 1.0) -> LogOddsField:
    """dxg.py:223-233 (O(n); same operation order as the fused device update)."""
    resid = np.asarray(col_marginal, dtype=float) - as_weights(c)
    delta = (1.0 - params.tau_mu * params.eta_mu) * mu.delta \
        + 4.0 * params.tau_mu * sup_norm * resid / np.asarray(c_tilde, dtype=float)
    return LogOddsField(delta)


def balance(mu: LogOddsField, beta: float) -> LogOddsField:
    """dxg.py:236-245."""
    if beta <= 0:
        raise ValueError("beta must be positive")
    return LogOddsField(np.clip(mu.delta, -beta, beta))


def _engine_for(kernel, r, c, params) -> DxgEngine:
    return DxgEngine(kernel, as_weights(r), as_weights(c), params, group=default_group())


# One cached engine for repeated dxg_step calls on the same (kernel, r, c, params):
# buffers stay allocated and, when the caller passes back the state the previous
# call returned, the row shifts of that sweep are reused (no row-max pass).
_STEP_CACHE: dict = {}


def dxg_step(state: DxgState, kernel: CostKernel, r: Histogram, c: Histogram, params: DxgParams,
             workers: int = 1) -> DxgState:
    """One extragradient iteration (dxg.py:261-279): one device sweep + fused O(n) update.

    Host state in, host state out: the state is copied H2D, iterated in HBM and
    copied back (the reference-facing call with host buffers).
    """
    kernel = _dev_kernel(kernel)
    key = (id(kernel), id(r), id(c), params)
    ent = _STEP_CACHE.get("entry")
    if ent is None or ent["key"] != key:
        _STEP_CACHE.clear()
        ent = {"key": key, "refs": (kernel, r, c), "eng": _engine_for(kernel, r, c, params), "last": None}
        _STEP_CACHE["entry"] = ent
    eng = ent["eng"]
    w = state.weights
    last = ent["last"]
    warm = (last is not None and (w.a, w.s, w.t) == last[2] and np.array_equal(state.mu.delta, last[0])
            and np.array_equal(w.b, last[1]))
    eng.load_state(state.mu.delta, w.b, w.a, w.s, w.t, keep_shift=warm)
    eng.sweep()
    eng.update()
    delta, b, a, s, t = eng.read_state()
    out = DxgState(LogOddsField(delta), TransportLogWeights(a=a, b=b, s=s, t=int(w.t) + 1))
    ent["last"] = (delta, b, (a, s, int(w.t) + 1))
    return out


def _plan_stats(state: TransportLogWeights, kernel: CostKernel, r: Histogram, workers: int = 1):
    """(<C, D_r p>, c(D_r p), H(D_r p)) in one device sweep (dxg.py:282-310)."""
    kernel = _dev_kernel(kernel)
    torch = _torch()
    dev = kernel.device
    rw = as_weights(r)
    r0, r1 = kernel.local_rows
    with torch.cuda.device(dev):
        bt = _to_dev(state.b, dev)
        w, keep = _wsets(dev, [(state.a, bt)])
        rt = _to_dev(rw, dev)
        col = torch.empty(kernel.n, dtype=torch.float64, device=dev)
        out3 = torch.zeros(3, dtype=torch.float64, device=dev)
        ws = _ws(kernel, 1, r1 - r0)
        _lib.check(_lib.lib().leanot_plan_stats(kernel.cost_struct(), r0, r1, C.byref(w), rt.data_ptr(),
                                                col.data_ptr(), out3.data_ptr(), ws.data_ptr(),
                                                _lib.stream_handle()), "plan_stats")
        cost, ent_rows, _ = out3.cpu().tolist()
        colh = col.cpu().numpy()
        del keep
    pos = rw > 0
    ent = ent_rows + float(-(rw[pos] * np.log(rw[pos])).sum())
    return cost, colh, ent


def primal_penalized_value(state: TransportLogWeights, kernel: CostKernel, r: Histogram, c: Histogram,
                           eta: float, workers: int = 1) -> float:
    """dxg.py:313-318."""
    kernel = _dev_kernel(kernel)
    cost, col, ent = _plan_stats(state, kernel, r, workers)
    pen = 2.0 * kernel.sup_norm * float(np.abs(col - as_weights(c)).sum())
    return cost + pen - eta * ent


def _row_reduce(kernel: CostKernel, v, mode: str, eta: float = 1.0):
    """Per-row min_j (C_ij + v_j) or LSE_j(-(C_ij + v_j)/eta) on device."""
    torch = _torch()
    dev = kernel.device
    r0, r1 = kernel.local_rows
    with torch.cuda.device(dev):
        vt = _to_dev(v, dev)
        out = torch.empty(r1 - r0, dtype=torch.float64, device=dev)
        L = _lib.lib()
        if mode == "min":
            _lib.check(L.leanot_row_min(kernel.cost_struct(), r0, r1, vt.data_ptr(), out.data_ptr(),
                                        _lib.stream_handle()), "row_min")
        else:
            _lib.check(L.leanot_row_lse_affine(kernel.cost_struct(), r0, r1, vt.data_ptr(), 1.0, -1.0 / eta,
                                               out.data_ptr(), _lib.stream_handle()), "row_lse")
        return out.cpu().numpy()


def dual_penalized_value(mu: LogOddsField, kernel: CostKernel, r: Histogram, c: Histogram, eta: float,
                         workers: int = 1) -> float:
    """dxg.py:321-349 (derivation sign inside the LSE)."""
    kernel = _dev_kernel(kernel)
    d = mu.diff()
    shift = 2.0 * kernel.sup_norm * d
    rw = as_weights(r)
    if eta > 0:
        red = _row_reduce(kernel, shift, "lse", eta)
        pos = rw > 0
        h_r = float(-(rw[pos] * np.log(rw[pos])).sum())
        inner = -eta * float(rw @ red) - eta * h_r
    else:
        red = _row_reduce(kernel, shift, "min")
        inner = float(rw @ red)
    return float(-2.0 * kernel.sup_norm * (as_weights(c) @ d) + inner)


def recover_eot_potentials(state: DxgState, mu: LogOddsField, kernel: CostKernel, r: Histogram, eta: float,
                           workers: int = 1) -> DualPotentials:
    """dxg.py:352-372."""
    if eta <= 0:
        raise ValueError("potential recovery requires eta > 0")
    rw = as_weights(r)
    if not bool(np.all(rw > 0)):
        raise ValueError("potential recovery requires full-support r")
    kernel = _dev_kernel(kernel)
    psi = -2.0 * kernel.sup_norm * mu.diff()
    log_z = _row_reduce(kernel, -psi, "lse", eta)   # LSE_j(-(C_ij - psi_j)/eta)
    phi = eta * (np.log(rw) - log_z)
    return DualPotentials(phi - phi.mean(), psi - psi.mean(), eta, converged=True, sweeps=state.weights.t)


def _evaluate(state: DxgState, kernel, r, c, eta, workers):
    """dxg.py:412-417 (standalone form; solve() folds it into its sweeps)."""
    cost, col, ent = _plan_stats(state.weights, kernel, r, workers)
    infeas = float(np.abs(col - as_weights(c)).sum())
    primal = cost + 2.0 * kernel.sup_norm * infeas - eta * ent
    dual = dual_penalized_value(state.mu, kernel, r, c, eta, workers)
    return primal, dual, infeas


def solve(kernel: CostKernel, r: Histogram, c: Histogram, params: DxgParams,
          termination: Termination = Termination(), log_stride: int = 25,
          workers: int = 1, dense_cap: int = DENSE_CAP) -> DxgSolution:
    """Run DXG with gap/infeasibility termination (dxg.py:420-472).

    The loop structure, logging points, termination test and returned record
    follow the reference.  Between logging points the iterations run as one
    CUDA graph (small n) or back-to-back launches, with no host sync.  With a
    timeout the wall clock is checked after every iteration, as in the
    reference (this forces one host sync per iteration).
    """
    rw, cw = as_weights(r), as_weights(c)
    if kernel.n != rw.size or kernel.n != cw.size:
        raise ValueError("kernel/marginal size mismatch")
    if params.alpha == 0.0 and not bool(np.all(cw > 0)):
        raise ValueError("alpha = 0 requires a full-support column marginal")
    kernel = _dev_kernel(kernel)
    torch = _torch()
    eng = DxgEngine(kernel, rw, cw, params, group=default_group())
    n = kernel.n
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    t0 = time.perf_counter()
    trajectory: list[TrajectoryPoint] = []
    converged = False
    it = 0
    swept = False          # plan->col holds the marginals of the current state
    max_iter = termination.max_iter
    timeout = termination.timeout

    def log_point():
        nonlocal swept
        if not swept:
            eng.sweep(evaluate=True)
            swept = True
        primal, dual, infeas = eng.evaluate()
        s_val = eng.last_scalars[2]      # read with the evaluation buffer (one transfer)
        point = TrajectoryPoint(it, time.perf_counter() - t0, primal, dual, primal - dual, infeas, s_val)
        trajectory.append(point)
        return point

    # small single-process plans: one launch per logging interval (update + iterations +
    # evaluation sweep, leanot_dxg_iterate_eval) and one device->host read
    folded = timeout is None and eng.world == 1 and n <= 1024
    while folded and it < max_iter:
        nxt = min(((it // log_stride) + 1) * log_stride, max_iter)
        with torch.cuda.device(eng.device):
            rc = _lib.lib().leanot_dxg_iterate_eval(C.byref(eng.plan), int(nxt - it), 1 if swept else 0,
                                                    _lib.stream_handle())
        if rc != _lib.LEANOT_OK:
            if it == 0 and not swept:
                folded = False          # not eligible (e.g. separable grid path): regular loop
                break
            _lib.check(rc, "dxg_iterate_eval")
        it = nxt
        swept = True
        primal, dual, infeas = eng.evaluate_buffer()
        point = TrajectoryPoint(it, time.perf_counter() - t0, primal, dual, primal - dual, infeas,
                                eng.last_scalars[2])
        trajectory.append(point)
        if point.gap <= termination.eps / 6.0 and point.col_infeas_l1 <= termination.eps / 6.0:
            converged = True
            break
    while not folded and it < max_iter:
        if timeout is None:
            # run to the next logging point without host syncs:
            # update (uses the swept marginals) + k x (sweep, update)
            nxt = min(((it // log_stride) + 1) * log_stride, max_iter)
            k = nxt - it
            if not swept:
                eng.sweep()
            eng.update()
            eng.iterate(k - 1)
            it = nxt
            swept = False
            timed_out = False
        else:
            if not swept:
                eng.sweep()
            eng.update()
            swept = False
            it += 1
            torch.cuda.synchronize(eng.device)
            timed_out = time.perf_counter() - t0 > timeout
            if eng.group is not None:   # every rank must take the same branch (collectives below)
                timed_out = any_rank(timed_out, eng.group)
        if it % log_stride == 0 or it == max_iter or timed_out:
            # the evaluation sweep is also the next iteration's sweep
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

    seconds = time.perf_counter() - t0
    colm = eng.col_now()               # column_marginal(state.weights) (dxg.py:464)
    report = infeasibility(colm, True, Histogram(cw) if isinstance(c, np.ndarray) else c)
    delta, b, a, s, t = eng.read_state()
    eng.close()
    state = DxgState(LogOddsField(delta), TransportLogWeights(a=a, b=b, s=s, t=it))
    sol = DxgSolution(state, converged, it, seconds, trajectory, report, workers=workers)
    if kernel.n <= dense_cap and _holds_all_rows(kernel):
        # materialize, Round (Alg. 1) and <C, pi> all on device (dxg.py:467-471).  A row shard
        # of a stored cost (multi-GPU runs) cannot materialize the n x n plan: no rounding then.
        P = round_on_device(_plan_on_device(state.weights, kernel, rw), rw, cw)
        out = torch.empty(1025, dtype=torch.float64, device=kernel.device)
        with torch.cuda.device(kernel.device):
            _lib.check(_lib.lib().leanot_plan_cost(kernel.cost_struct(), P.data_ptr(), kernel.n, out[1024:].data_ptr(),
                                                   out.data_ptr(), _lib.stream_handle()), "plan_cost")
        sol.rounded_plan = DenseCoupling(P.cpu().numpy())
        sol.rounded_cost = float(out[1024].item())
    return sol


# ---------------------------------------------------------------------------
# dense PDXG reference (dxg.py:480-521) -- equivalence oracle, dense, n <= cap
# ---------------------------------------------------------------------------


@dataclass
class PdxgState:
    mu: LogOddsField
    log_p: np.ndarray


def pdxg_init(n: int, cap: int = DENSE_CAP) -> PdxgState:
    if n > cap:
        raise ValueError("dense reference limited to the dense cap")
    return PdxgState(LogOddsField.uniform(n), np.full((n, n), -math.log(n)))


def pdxg_reference_step(state: PdxgState, kernel: CostKernel, r: Histogram, c: Histogram,
                        params: DxgParams) -> PdxgState:
    """Dense extragradient step (dxg.py:494-521) on device: the row updates
    z = decay log_p - tau (C + 2 sup d) minus their row LSEs (`leanot_pdxg_rows`, the cost
    evaluated on device as in the sweeps) and the column marginals r @ exp(.)
    (`leanot_pdxg_colsum`); the O(n) dual steps are the host functions above."""
    kernel = _dev_kernel(kernel)
    torch = _torch()
    n = kernel.n
    if state.log_p.shape != (n, n):
        raise ValueError("state/kernel size mismatch")
    if not _holds_all_rows(kernel):
        raise ValueError("the dense reference step needs every row of the cost")
    dev = kernel.device
    cw = as_weights(c)
    c_tilde = cw + params.alpha / n
    sup = kernel.sup_norm
    decay = 1.0 - params.tau_p * params.eta
    lib = _lib.lib()
    with torch.cuda.device(dev):
        s = _lib.stream_handle()
        lp = torch.from_numpy(np.ascontiguousarray(state.log_p, dtype=float)).to(dev)
        rt = _to_dev(as_weights(r), dev)
        col = torch.empty(n, dtype=torch.float64, device=dev)

        def colsum(M):
            _lib.check(lib.leanot_pdxg_colsum(M.data_ptr(), n, n, rt.data_ptr(), col.data_ptr(), s), "pdxg_colsum")
            return col.cpu().numpy()

        def rows(dvec, out):
            d = _to_dev(np.ascontiguousarray(dvec, dtype=float), dev)
            _lib.check(lib.leanot_pdxg_rows(kernel.cost_struct(), lp.data_ptr(), n, decay, params.tau_p, 2.0 * sup,
                                            d.data_ptr(), out.data_ptr(), s), "pdxg_rows")
            return out

        col_now = colsum(lp)
        mu_bar = dual_md_step(state.mu, col_now, Histogram(cw), c_tilde, params, sup)
        buf = torch.empty_like(lp)
        col_bar = colsum(rows(state.mu.diff(), buf))
        mu_next = balance(dual_md_step(state.mu, col_bar, Histogram(cw), c_tilde, params, sup), params.beta)
        lpn = rows(mu_bar.diff(), buf).cpu().numpy()
    return PdxgState(mu_next, lpn)
