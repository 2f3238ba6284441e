"""CPU oracle for the DXG hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference solver's algorithm
(`leanot`, /root/reference/pkg/src/leanot/*.py).  It exists so that tests,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` have a checker that runs on any host (the reference itself is not
present on the GPU box).  The product path (`paper_2511_11359_b200`) never
imports it.

Pinning: the restatement is checked against golden vectors produced by running
the reference in the build container (`oracle/gen_golden.py` ->
`tests/golden/*.npz`, see tests/test_oracle_golden.py).  Block structure
(128-row blocks, max-shifted softmax, block-ordered accumulation) follows the
reference so that the oracle reproduces it to the last few ulps.

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

BLOCK_ROWS = 128          # core.py:44
SIMPLEX_ATOL = 1e-12      # core.py:46
MASS_EPS = 1e-15          # rounding.py:20

# ---------------------------------------------------------------------------
# cost providers (core.py:167-288) -- each exposes n, scale, sup_norm, block()
# ---------------------------------------------------------------------------


class DenseCost:
    """ExplicitKernel restated (core.py:239-261): normalized copy of a matrix."""

    def __init__(self, m):
        m = np.asarray(m, dtype=float)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("explicit cost matrix must be square")
        if np.any(m < 0):
            raise ValueError("cost entries must be nonnegative")
        self.n = m.shape[0]
        sup = float(m.max()) if m.size else 0.0
        self.scale = sup if sup > 0 else 1.0
        self.sup_norm = 1.0 if sup > 0 else 0.0
        self.m = m / self.scale

    def block(self, i0, i1):
        return self.m[i0:i1]


class GridCost:
    """GridKernel restated (core.py:200-236)."""

    def __init__(self, height, width, p=2):
        if height < 1 or width < 1 or p not in (1, 2, 3):
            raise ValueError("bad grid")
        self.height, self.width, self.p = int(height), int(width), int(p)
        self.n = self.height * self.width
        sup = float((self.height - 1) ** p + (self.width - 1) ** p)
        self.scale = sup if sup > 0 else 1.0
        self.sup_norm = 1.0 if sup > 0 else 0.0
        k = np.arange(self.n)
        self.rows = (k // self.width).astype(float)
        self.cols = (k % self.width).astype(float)

    def block(self, i0, i1):
        dr = np.abs(self.rows[i0:i1, None] - self.rows[None, :])
        dc = np.abs(self.cols[i0:i1, None] - self.cols[None, :])
        if self.p == 1:
            out = dr + dc
        elif self.p == 2:
            out = dr * dr + dc * dc
        else:
            out = dr ** 3 + dc ** 3
        return out / self.scale


class PointCost:
    """ColorKernel restated (core.py:264-288); `scale` may be supplied when it
    is known by construction (skips the O(n^2 d) max pass, core.py:279-282)."""

    def __init__(self, features, p=2, scale=None):
        f = np.asarray(features, dtype=float)
        if f.ndim != 2 or p not in (1, 2, 3):
            raise ValueError("bad features")
        self.f, self.p, self.n = f, int(p), f.shape[0]
        if scale is None:
            sup = 0.0
            for i0 in range(0, self.n, BLOCK_ROWS):
                i1 = min(i0 + BLOCK_ROWS, self.n)
                d = np.abs(f[i0:i1, None, :] - f[None, :, :]) ** p
                sup = max(sup, float(d.sum(axis=2).max()))
        else:
            sup = float(scale)
        self.scale = sup if sup > 0 else 1.0
        self.sup_norm = 1.0 if sup > 0 else 0.0

    def block(self, i0, i1):
        d = np.abs(self.f[i0:i1, None, :] - self.f[None, :, :]) ** self.p
        return d.sum(axis=2) / self.scale


# Counter-based generator for the stored-C benchmark instance:
# C_ij = U[0,1) from splitmix64(seed, i, j); entry (0, n-1) is forced to 1.0 so the
# sup-norm is 1 by construction (scale = 1, normalization is the identity).
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def hash_u01(seed: int, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer of key=(i<<32|j) ^ seed*golden, top 53 bits -> [0,1)."""
    with np.errstate(over="ignore"):
        key = (rows.astype(np.uint64)[:, None] << np.uint64(32)) | cols.astype(np.uint64)[None, :]
        z = key ^ (np.uint64(seed) * _GOLDEN)
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


class HashCost:
    """Stored-C benchmark matrix regenerated block by block on the host."""

    def __init__(self, n, seed=0):
        self.n, self.seed = int(n), int(seed)
        self.scale, self.sup_norm = 1.0, 1.0
        self._cols = np.arange(self.n)

    def block(self, i0, i1):
        out = hash_u01(self.seed, np.arange(i0, i1), self._cols)
        if i0 == 0 and self.n > 1:
            out[0, self.n - 1] = 1.0
        return out


# ---------------------------------------------------------------------------
# scheduling (core.py:291-309)
# ---------------------------------------------------------------------------


def row_blocks(n, block_rows=BLOCK_ROWS):
    return [(i0, min(i0 + block_rows, n)) for i0 in range(0, n, block_rows)]


def run_blocks(fn, n, workers=1, block_rows=BLOCK_ROWS):
    """Results in block order regardless of worker count (core.py:297-309)."""
    ranges = row_blocks(n, block_rows)
    if workers <= 1 or len(ranges) == 1:
        return [fn(i0, i1) for i0, i1 in ranges]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(lambda ab: fn(*ab), ranges))


def lse_rows(z):
    """core.py:67-70."""
    m = z.max(axis=1)
    return m + np.log(np.exp(z - m[:, None]).sum(axis=1))


def normalized_hist(raw):
    """Histogram.normalized (core.py:130-137) without the dataclass."""
    raw = np.asarray(raw, dtype=float).ravel()
    return raw / raw.sum()


def check_hist(w):
    """Histogram.__post_init__ validation (core.py:119-128)."""
    w = np.asarray(w, dtype=float).ravel()
    if w.size == 0 or np.any(w < 0) or abs(w.sum() - 1.0) > SIMPLEX_ATOL:
        raise ValueError("not a histogram")
    return w


# ---------------------------------------------------------------------------
# DXG (dxg.py)
# ---------------------------------------------------------------------------


@dataclass
class Params:
    """DxgParams (dxg.py:100-128)."""
    eta: float
    eta_mu: float
    tau_p: float
    tau_mu: float
    beta: float
    alpha: float


def params_tuned(eta=0.0, **over):
    """dxg.py:131-133 (+ with_overrides, dxg.py:127-128)."""
    p = Params(eta=eta, eta_mu=0.0, tau_p=1.0, tau_mu=1.0, beta=1.1, alpha=0.01)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def params_loose(n, eps, min_marginal, cost_sup=1.0):
    """dxg.py:157-172."""
    eta = min(cost_sup / (-math.log(min_marginal)), eps / (16.0 * math.log(n)))
    tau_mu = 1.0 / (4.0 * math.sqrt(n))
    min_ct = min_marginal + 1.0 / n
    tau_p = min_ct / (n ** -0.5 + eta * min_ct)
    eta_mu = min(eps / (16.0 * math.log(2.0)), eta * tau_p / tau_mu)
    return Params(eta, eta_mu, tau_p, tau_mu, math.log(3.0), 1.0)


@dataclass
class Iterate:
    """DxgState = (LogOddsField, TransportLogWeights) (dxg.py:57-97, 175-182)."""
    delta: np.ndarray
    a: float
    b: np.ndarray
    s: float
    t: int

    @classmethod
    def zero(cls, n):
        return cls(np.zeros(n), 0.0, np.zeros(n), 0.0, 0)

    def copy(self):
        return Iterate(self.delta.copy(), self.a, self.b.copy(), self.s, self.t)


def _softmax_block(a, b, Cb):
    """Rows of the implicit plan for one block (dxg.py:199-202)."""
    z = -(a * Cb + b[None, :])
    z -= z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


def column_marginals(cost, r, weight_sets, workers=1):
    """One streamed pass producing c(D_r p) for several (a, b) weight sets.

    Per weight set this is exactly column_marginal (dxg.py:193-208); sharing
    the block of C between weight sets is the fused-iteration restructuring of
    SURVEY.md §0.3 (both half-step marginals depend only on the current state).
    """
    def work(i0, i1):
        Cb = cost.block(i0, i1)
        return [r[i0:i1] @ _softmax_block(a, b, Cb) for a, b in weight_sets]

    cols = [np.zeros(cost.n) for _ in weight_sets]
    for parts in run_blocks(work, cost.n, workers):
        for acc, part in zip(cols, parts):
            acc += part
    return cols


def _mirror(delta, col, c, c_tilde, prm, sup):
    """dual_md_step (dxg.py:223-233)."""
    resid = np.asarray(col, dtype=float) - c
    return (1.0 - prm.tau_mu * prm.eta_mu) * delta \
        + 4.0 * prm.tau_mu * sup * resid / np.asarray(c_tilde, dtype=float)


def _advance(a, b, s, t, diff, prm, sup):
    """_advance_weights (dxg.py:248-258)."""
    decay = 1.0 - prm.tau_p * prm.eta
    nb = decay * b + 2.0 * prm.tau_p * sup * diff
    nb -= nb.max()
    return decay * a + prm.tau_p, nb, decay * s + prm.tau_p * prm.eta, t + 1


def step(it: Iterate, cost, r, c, prm: Params, workers=1, return_cols=False):
    """dxg_step (dxg.py:261-279), both column marginals from one sweep."""
    n = cost.n
    c_tilde = c + prm.alpha / n
    sup = cost.sup_norm
    a_bar, b_bar, s_bar, t_bar = _advance(it.a, it.b, it.s, it.t, np.tanh(0.5 * it.delta), prm, sup)
    col_now, col_bar = column_marginals(cost, r, [(it.a, it.b), (a_bar, b_bar)], workers)
    delta_bar = _mirror(it.delta, col_now, c, c_tilde, prm, sup)
    delta_next = np.clip(_mirror(it.delta, col_bar, c, c_tilde, prm, sup), -prm.beta, prm.beta)
    a, b, s, t = _advance(it.a, it.b, it.s, it.t, np.tanh(0.5 * delta_bar), prm, sup)
    out = Iterate(delta_next, a, b, s, t)
    if return_cols:
        return out, col_now, col_bar
    return out


def plan_stats(a, b, cost, r, workers=1):
    """_plan_stats (dxg.py:282-310): (<C, D_r p>, c(D_r p), H(D_r p))."""
    def work(i0, i1):
        Cb = cost.block(i0, i1)
        z = -(a * Cb + b[None, :])
        m = z.max(axis=1, keepdims=True)
        e = np.exp(z - m)
        ssum = e.sum(axis=1, keepdims=True)
        p = e / ssum
        rb = r[i0:i1]
        cst = float((rb[:, None] * p * Cb).sum())
        col = rb @ p
        plogp = (p * ((z - m) - np.log(ssum))).sum(axis=1)
        return cst, col, float(-(rb * plogp).sum())

    cost_v, ent = 0.0, 0.0
    col = np.zeros(cost.n)
    for pc, pcol, pe in run_blocks(work, cost.n, workers):
        cost_v += pc
        col += pcol
        ent += pe
    pos = r > 0
    ent += float(-(r[pos] * np.log(r[pos])).sum())
    return cost_v, col, ent


def dual_value(delta, cost, r, c, eta, workers=1):
    """dual_penalized_value (dxg.py:321-349)."""
    d = np.tanh(0.5 * delta)
    shift = 2.0 * cost.sup_norm * d
    if eta > 0:
        red = np.concatenate(run_blocks(
            lambda i0, i1: lse_rows(-(cost.block(i0, i1) + shift[None, :]) / eta), cost.n, workers))
        pos = r > 0
        h_r = float(-(r[pos] * np.log(r[pos])).sum())
        inner = -eta * float(r @ red) - eta * h_r
    else:
        red = np.concatenate(run_blocks(
            lambda i0, i1: (cost.block(i0, i1) + shift[None, :]).min(axis=1), cost.n, workers))
        inner = float(r @ red)
    return float(-2.0 * cost.sup_norm * (c @ d) + inner)


def evaluate(it: Iterate, cost, r, c, eta, workers=1):
    """_evaluate (dxg.py:412-417) -> (primal, dual, infeas, col)."""
    cst, col, ent = plan_stats(it.a, it.b, cost, r, workers)
    infeas = float(np.abs(col - c).sum())
    primal = cst + 2.0 * cost.sup_norm * infeas - eta * ent
    return primal, dual_value(it.delta, cost, r, c, eta, workers), infeas, col


def solve(cost, r, c, prm, eps=1e-10, max_iter=1_000_000, log_stride=25, workers=1,
          callback=None):
    """solve (dxg.py:420-472) without timeout and without dense rounding.

    Returns (iterate, converged, iterations, trajectory[(iter, primal, dual, gap,
    infeas, s)], final column marginal).
    """
    if cost.n != r.size or cost.n != c.size:
        raise ValueError("kernel/marginal size mismatch")
    it = Iterate.zero(cost.n)
    traj, k, converged, col = [], 0, False, None
    while k < max_iter:
        it = step(it, cost, r, c, prm, workers)
        k += 1
        if k % log_stride == 0 or k == max_iter:
            primal, dual, infeas, col = evaluate(it, cost, r, c, prm.eta, workers)
            traj.append((k, primal, dual, primal - dual, infeas, it.s))
            if callback:
                callback(k, traj[-1])
            if primal - dual <= eps / 6.0 and infeas <= eps / 6.0:
                converged = True
                break
    if not traj or traj[-1][0] != k:
        primal, dual, infeas, col = evaluate(it, cost, r, c, prm.eta, workers)
        traj.append((k, primal, dual, primal - dual, infeas, it.s))
    return it, converged, k, traj, col


def recover_potentials(delta, cost, r, eta, workers=1):
    """recover_eot_potentials (dxg.py:352-372) -> (phi, psi), mean-centered."""
    psi = -2.0 * cost.sup_norm * np.tanh(0.5 * delta)
    log_z = np.concatenate(run_blocks(
        lambda i0, i1: lse_rows(-(cost.block(i0, i1) - psi[None, :]) / eta), cost.n, workers))
    phi = eta * (np.log(r) - log_z)
    return phi - phi.mean(), psi - psi.mean()


def pdxg_step(delta, log_p, C, r, c, prm, sup):
    """Dense PDXG reference (dxg.py:494-521), independent of the implicit plan."""
    n = C.shape[0]
    c_tilde = c + prm.alpha / n
    decay = 1.0 - prm.tau_p * prm.eta
    col_now = r @ np.exp(log_p)
    delta_bar = _mirror(delta, col_now, c, c_tilde, prm, sup)
    lp_bar = decay * log_p - prm.tau_p * (C + 2.0 * sup * np.tanh(0.5 * delta)[None, :])
    lp_bar -= lse_rows(lp_bar)[:, None]
    col_bar = r @ np.exp(lp_bar)
    delta_next = np.clip(_mirror(delta, col_bar, c, c_tilde, prm, sup), -prm.beta, prm.beta)
    lp_next = decay * log_p - prm.tau_p * (C + 2.0 * sup * np.tanh(0.5 * delta_bar)[None, :])
    lp_next -= lse_rows(lp_next)[:, None]
    return delta_next, lp_next


# ---------------------------------------------------------------------------
# barycenter (barycenter.py)
# ---------------------------------------------------------------------------


@dataclass
class BaryIterate:
    """BarycenterState (barycenter.py:44-75)."""
    deltas: np.ndarray
    bs: np.ndarray
    a: float
    s: float
    t: int
    w: np.ndarray
    eta: float

    @classmethod
    def zero(cls, n, weights, eta):
        w = np.asarray(weights, dtype=float).ravel()
        w = w / w.sum()
        m = w.size
        return cls(np.zeros((m, n)), np.zeros((m, n)), 0.0, 0.0, 0, w, eta)


def log_normalizers(a, bs, cost, workers=1):
    """_log_normalizers (barycenter.py:78-87): (m, n) LSE_j(-(a C_ij + b_kj))."""
    out = np.empty_like(bs)
    for k in range(bs.shape[0]):
        out[k] = np.concatenate(run_blocks(
            lambda i0, i1, bk=bs[k]: lse_rows(-(a * cost.block(i0, i1) + bk[None, :])), cost.n, workers))
    return out


def marginal_from_logz(w, log_z):
    """_marginal_from_logz (barycenter.py:90-97): sorted k-sum, max shift, normalize."""
    g = np.sort(w[:, None] * log_z, axis=0).sum(axis=0)
    g -= g.max()
    e = np.exp(g)
    return e / e.sum()


def bary_step(st: BaryIterate, cost, marginals, prm, workers=1):
    """dxgb_step (barycenter.py:108-151)."""
    m, n = st.deltas.shape
    sup = cost.sup_norm
    decay = 1.0 - prm.tau_p * prm.eta
    a_next = decay * st.a + prm.tau_p
    s_next = decay * st.s + prm.tau_p * prm.eta
    r_now = marginal_from_logz(st.w, log_normalizers(st.a, st.bs, cost, workers))
    deltas_bar = np.empty_like(st.deltas)
    bs_bar = np.empty_like(st.bs)
    for k in range(m):
        ct = marginals[k] + prm.alpha / n
        (col_now,) = column_marginals(cost, r_now, [(st.a, st.bs[k])], workers)
        deltas_bar[k] = _mirror(st.deltas[k], col_now, marginals[k], ct, prm, sup)
        b = decay * st.bs[k] + 2.0 * prm.tau_p * sup * np.tanh(0.5 * st.deltas[k])
        bs_bar[k] = b - b.max()
    r_bar = marginal_from_logz(st.w, log_normalizers(a_next, bs_bar, cost, workers))
    deltas_next = np.empty_like(st.deltas)
    bs_next = np.empty_like(st.bs)
    for k in range(m):
        ct = marginals[k] + prm.alpha / n
        (col_bar,) = column_marginals(cost, r_bar, [(a_next, bs_bar[k])], workers)
        deltas_next[k] = np.clip(_mirror(st.deltas[k], col_bar, marginals[k], ct, prm, sup),
                                 -prm.beta, prm.beta)
        b = decay * st.bs[k] + 2.0 * prm.tau_p * sup * np.tanh(0.5 * deltas_bar[k])
        bs_next[k] = b - b.max()
    return BaryIterate(deltas_next, bs_next, a_next, s_next, st.t + 1, st.w, st.eta)


def bary_dual(st: BaryIterate, cost, marginals, workers=1):
    """_bary_dual_value (barycenter.py:172-195)."""
    eta, sup = st.eta, cost.sup_norm
    m, n = st.deltas.shape
    log_z = np.empty((m, n))
    lead = 0.0
    for k in range(m):
        d = np.tanh(0.5 * st.deltas[k])
        shift = 2.0 * sup * d
        log_z[k] = np.concatenate(run_blocks(
            lambda i0, i1, sh=shift: lse_rows(-(cost.block(i0, i1) + sh[None, :]) / eta), cost.n, workers))
        lead += st.w[k] * (-2.0 * sup * float(marginals[k] @ d))
    g = (st.w[:, None] * log_z).sum(axis=0)
    gm = g.max()
    return lead - eta * (gm + float(np.log(np.exp(g - gm).sum())))


def bary_evaluate(st: BaryIterate, cost, marginals, workers=1):
    """_bary_evaluate (barycenter.py:214-224) -> (primal, dual, infeas[m], r)."""
    r = marginal_from_logz(st.w, log_normalizers(st.a, st.bs, cost, workers))
    primal = 0.0
    infeas = np.empty(len(marginals))
    for k in range(len(marginals)):
        cst, col, ent = plan_stats(st.a, st.bs[k], cost, r, workers)
        infeas[k] = float(np.abs(col - marginals[k]).sum())
        primal += st.w[k] * (cst + 2.0 * sup_of(cost) * infeas[k] - st.eta * ent)
    return primal, bary_dual(st, cost, marginals, workers), infeas, r


def sup_of(cost):
    return cost.sup_norm


def bary_solve(cost, marginals, w, prm, eps=1e-10, max_iter=1_000_000, log_stride=25, workers=1):
    """dxgb_solve (barycenter.py:227-277) without timeout."""
    st = BaryIterate.zero(cost.n, w, prm.eta)
    traj, k, converged = [], 0, False
    while k < max_iter:
        st = bary_step(st, cost, marginals, prm, workers)
        k += 1
        if k % log_stride == 0 or k == max_iter:
            primal, dual, infeas, _ = bary_evaluate(st, cost, marginals, workers)
            traj.append((k, primal, dual, primal - dual, float(infeas.max()), st.s))
            if primal - dual <= eps / 6.0 and float(infeas.max()) <= eps / 6.0:
                converged = True
                break
    if not traj or traj[-1][0] != k:
        primal, dual, infeas, _ = bary_evaluate(st, cost, marginals, workers)
        traj.append((k, primal, dual, primal - dual, float(infeas.max()), st.s))
    r = marginal_from_logz(st.w, log_normalizers(st.a, st.bs, cost, workers))
    return st, converged, k, traj, r


# ---------------------------------------------------------------------------
# rounding (rounding.py:63-98)
# ---------------------------------------------------------------------------


def round_to_polytope(m, r, c):
    """Alg. 1 Round (rounding.py:63-87)."""
    row = m.sum(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        x = np.where(row > 0, np.minimum(r / row, 1.0), 1.0)
    m = m * x[:, None]
    col = m.sum(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.where(col > 0, np.minimum(c / col, 1.0), 1.0)
    m = m * y[None, :]
    dr = r - m.sum(axis=1)
    dc = c - m.sum(axis=0)
    mass = dr.sum()
    if mass > MASS_EPS:
        m = m + np.outer(dr, dc) / mass
    return m


def default_workers():
    return max(1, len(os.sched_getaffinity(0)))


# ---------------------------------------------------------------------------
# Sinkhorn / IBP baselines (sinkhorn.py) -- SURVEY.md §8f item 1
# ---------------------------------------------------------------------------


def col_lse(cost, phi, eta, workers=1):
    """_col_lse (sinkhorn.py:47-62): LSE_i((phi_i - C_ij)/eta), block-merged running max/sum."""
    n = cost.n
    run_m = np.full(n, -np.inf)
    run_s = np.zeros(n)

    def work(i0, i1):
        z = (phi[i0:i1, None] - cost.block(i0, i1)) / eta
        m = z.max(axis=0)
        return m, np.exp(z - m[None, :]).sum(axis=0)

    for m, s in run_blocks(work, n, workers):
        new_m = np.maximum(run_m, m)
        run_s = run_s * np.exp(run_m - new_m) + s * np.exp(m - new_m)
        run_m = new_m
    return run_m + np.log(run_s)


def row_lse(cost, psi, eta, workers=1):
    """_row_lse (sinkhorn.py:65-71): LSE_j((psi_j - C_ij)/eta)."""
    return np.concatenate(run_blocks(lambda i0, i1: lse_rows((psi[None, :] - cost.block(i0, i1)) / eta),
                                     cost.n, workers))


def sinkhorn(cost, r, c, eta, tol=1e-9, max_iter=100_000, workers=1):
    """sinkhorn_solve (sinkhorn.py:74-110) -> (phi, psi, converged, sweeps, col_gap), centered."""
    log_r, log_c = np.log(r), np.log(c)
    psi = np.zeros(cost.n)
    best = None
    for sweep in range(1, max_iter + 1):
        phi = eta * log_r - eta * row_lse(cost, psi, eta, workers)
        psi_new = eta * log_c - eta * col_lse(cost, phi, eta, workers)
        gap = float(np.abs(c * np.expm1((psi - psi_new) / eta)).sum())
        if best is None or gap < best[4]:
            best = (phi, psi, True, sweep, gap)
        if gap <= tol:
            sh = phi.mean()
            return phi - sh, psi + sh, True, sweep, gap
        psi = psi_new
    phi, psi, _, sweep, gap = best
    sh = phi.mean()
    return phi - sh, psi + sh, False, sweep, gap


def eot_dual(phi, psi, eta, cost, r, c, workers=1):
    """eot_dual_value (sinkhorn.py:120-136)."""
    run_m, run_s = -np.inf, 0.0
    for m, s in run_blocks(lambda i0, i1: _blk_lse(phi, psi, eta, cost, i0, i1), cost.n, workers):
        new_m = max(run_m, m)
        run_s = run_s * np.exp(run_m - new_m) + s * np.exp(m - new_m)
        run_m = new_m
    return float(phi @ r + psi @ c - eta * (run_m + np.log(run_s)))


def _blk_lse(phi, psi, eta, cost, i0, i1):
    z = (phi[i0:i1, None] + psi[None, :] - cost.block(i0, i1)) / eta
    m = z.max()
    return m, np.exp(z - m).sum()


def sinkhorn_col(phi, psi, eta, cost, workers=1):
    """sinkhorn_column_marginal (sinkhorn.py:139-150)."""
    col = np.zeros(cost.n)
    for part in run_blocks(lambda i0, i1: np.exp((phi[i0:i1, None] + psi[None, :] - cost.block(i0, i1)) / eta)
                           .sum(axis=0), cost.n, workers):
        col += part
    return col / col.sum()


def ibp(cost, margs, weights, eta, tol=1e-9, max_iter=10_000, workers=1):
    """ibp_barycenter (sinkhorn.py:174-228) -> (bary, phis, psis, converged, sweeps, gap, log_r)."""
    m, n = len(margs), cost.n
    w = np.asarray(weights, dtype=float).ravel()
    w = w / w.sum()
    log_c = np.stack([np.log(h) for h in margs])
    phis, psis = np.zeros((m, n)), np.zeros((m, n))
    log_r = np.full(n, -np.log(n))
    gap, converged, sweeps = np.inf, False, 0
    for sweeps in range(1, max_iter + 1):
        psis_new = np.empty_like(psis)
        gaps = np.empty(m)
        for k in range(m):
            psis_new[k] = eta * log_c[k] - eta * col_lse(cost, phis[k], eta, workers)
            gaps[k] = np.abs(np.exp(log_c[k]) * np.expm1((psis[k] - psis_new[k]) / eta)).sum()
        gap = float(gaps.max())
        if sweeps > 1 and gap <= tol:
            converged = True
            break
        psis = psis_new
        row_lses = np.stack([row_lse(cost, psis[k], eta, workers) for k in range(m)])
        log_r = (w[:, None] * (phis / eta + row_lses)).sum(axis=0)
        phis = eta * log_r[None, :] - eta * row_lses
    bary = np.exp(log_r - log_r.max())
    return bary / bary.sum(), phis, psis, converged, sweeps, gap, log_r
