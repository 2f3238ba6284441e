"""Log-domain Sinkhorn and IBP on B200 -- drop-in for leanot.sinkhorn.

Same names, arguments and result types as the reference
(/root/reference/pkg/src/leanot/sinkhorn.py).  Every n^2 reduction (row LSE,
column LSE) runs in the sm_100a sweep kernels of libleanot_b200.so; the O(n)
potential updates and gap reductions are fused device kernels.  The host reads
one scalar (the column gap) per sweep, as the reference's stopping rule needs.
`DualPotentials` is also the result type of dxg.recover_eot_potentials.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import DENSE_CAP, Histogram, as_device_kernel, as_weights

__all__ = ["DualPotentials", "IbpResult", "sinkhorn_solve", "eot_dual_value", "sinkhorn_plan_dense",
           "sinkhorn_column_marginal", "ibp_barycenter", "ibp_plan_dense"]


@dataclass
class DualPotentials:
    """sinkhorn.py:30-44."""

    phi: np.ndarray
    psi: np.ndarray
    eta: float
    converged: bool = True
    sweeps: int = 0
    col_gap: float = field(default=np.nan)


@dataclass
class IbpResult:
    """sinkhorn.py:162-171."""

    barycenter: Histogram
    phis: np.ndarray
    psis: np.ndarray
    eta: float
    converged: bool
    sweeps: int
    col_gap: float
    log_r: np.ndarray = field(repr=False, default=None)


def _torch():
    import torch
    return torch


class _Sweeper:
    """Device workspaces for row/column LSE sweeps of one kernel.

    GridKernel costs take the separable O(n^1.5) path (two 1-D LSE convolutions per sweep,
    on the FP64 tensor cores while exp(-C/eta) stays representable); C is symmetric there,
    so the column LSE is the row LSE of the other potential."""

    def __init__(self, kernel, batch: int = 1):
        torch = _torch()
        self.k = kernel
        self.dev = kernel.device
        self.n = kernel.n
        self.cs = kernel.cost_struct()
        L = _lib.lib()
        self.sep = (self.cs.kind == _lib.COST_GRID and kernel.local_rows == (0, self.n)
                    and os.environ.get("LEANOT_GRID_SEPARABLE", "1") != "0")
        self.batch = int(batch)
        size = (L.leanot_grid_sep_lse_eta_ws_doubles(self.cs, self.batch) if self.sep
                else L.leanot_col_lse_ws_doubles(self.n, self.n))
        self.ws = torch.empty(int(size), dtype=torch.float64, device=self.dev)

    def vec(self, x=None):
        torch = _torch()
        if x is None:
            return torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=float)), device=self.dev)

    def row_lse(self, psi, eta, out):
        """LSE_j((psi_j - C_ij)/eta) (sinkhorn.py:65-71)."""
        if self.sep:
            self._sep_lse(psi, 1, eta, out)
            return
        _lib.check(_lib.lib().leanot_row_lse_affine(self.cs, 0, self.n, psi.data_ptr(), -1.0, 1.0 / eta,
                                                    out.data_ptr(), _lib.stream_handle()), "row_lse")

    def col_lse(self, phi, eta, out):
        """LSE_i((phi_i - C_ij)/eta) (sinkhorn.py:47-62)."""
        if self.sep:
            self._sep_lse(phi, 1, eta, out)
            return
        _lib.check(_lib.lib().leanot_col_lse(self.cs, 0, self.n, phi.data_ptr(), float(eta), out.data_ptr(),
                                             self.ws.data_ptr(), _lib.stream_handle()), "col_lse")

    def _sep_lse(self, v, nz, eta, out):
        """LSE_j((v_z,j - C_ij)/eta) for nz contiguous potentials (separable grid sweep)."""
        _lib.check(_lib.lib().leanot_grid_sep_lse_eta(self.cs, v.data_ptr(), int(nz), self.n, float(eta),
                                                      out.data_ptr(), self.n, self.ws.data_ptr(),
                                                      _lib.stream_handle()), "grid_sep_lse_eta")

    def row_lse_all(self, V, eta, OUT):
        """row_lse of every row of V (m x n, contiguous) into OUT (m x n)."""
        if self.sep and V.shape[0] <= self.batch:
            self._sep_lse(V, V.shape[0], eta, OUT)
            return
        for k in range(V.shape[0]):
            self.row_lse(V[k], eta, OUT[k])

    def col_lse_all(self, V, eta, OUT):
        """col_lse of every row of V (m x n, contiguous) into OUT (m x n)."""
        if self.sep and V.shape[0] <= self.batch:
            self._sep_lse(V, V.shape[0], eta, OUT)   # C symmetric on a grid
            return
        for k in range(V.shape[0]):
            self.col_lse(V[k], eta, OUT[k])


def _centered(pot: DualPotentials) -> DualPotentials:
    """sinkhorn.py:113-117."""
    shift = pot.phi.mean()
    pot.phi = pot.phi - shift
    pot.psi = pot.psi + shift
    return pot


def sinkhorn_solve(kernel, r, c, eta: float, tol: float = 1e-9, max_iter: int = 100_000,
                   workers: int = 1) -> DualPotentials:
    """Alternate exact row/column LSE updates until the column gap falls below tol (sinkhorn.py:74-110)."""
    if eta <= 0:
        raise ValueError("sinkhorn requires eta > 0")
    rw, cw = as_weights(r), as_weights(c)
    if not (bool(np.all(rw > 0)) and bool(np.all(cw > 0))):
        raise ValueError("sinkhorn requires full-support marginals")
    kernel = as_device_kernel(kernel)
    torch = _torch()
    L = _lib.lib()
    with torch.cuda.device(kernel.device):
        sw = _Sweeper(kernel)
        n = sw.n
        rt, ct = sw.vec(rw), sw.vec(cw)
        psi, psi_new, phi, lrow, lcol = sw.vec(), sw.vec(), sw.vec(), sw.vec(), sw.vec()
        best_phi, best_psi = sw.vec(), sw.vec()
        gap_t = torch.zeros(1, dtype=torch.float64, device=kernel.device)
        best = None
        s = _lib.stream_handle()
        for sweep in range(1, max_iter + 1):
            sw.row_lse(psi, eta, lrow)
            _lib.check(L.leanot_eta_log_minus(rt.data_ptr(), lrow.data_ptr(), float(eta), n, phi.data_ptr(), s),
                       "phi")
            sw.col_lse(phi, eta, lcol)
            _lib.check(L.leanot_sinkhorn_psi(ct.data_ptr(), lcol.data_ptr(), psi.data_ptr(), float(eta), n,
                                             psi_new.data_ptr(), gap_t.data_ptr(), s), "psi")
            gap = float(gap_t.item())
            if best is None or gap < best[1]:
                best_phi.copy_(phi)
                best_psi.copy_(psi)
                best = (sweep, gap)
            if gap <= tol:
                return _centered(DualPotentials(phi.cpu().numpy(), psi.cpu().numpy(), eta, True, sweep, gap))
            psi, psi_new = psi_new, psi
        out = _centered(DualPotentials(best_phi.cpu().numpy(), best_psi.cpu().numpy(), eta, True, best[0], best[1]))
        out.converged = False
        return out


def eot_dual_value(pot: DualPotentials, kernel, r, c, workers: int = 1) -> float:
    """<phi, r> + <psi, c> - eta * LSE_ij(-(C_ij - phi_i - psi_j)/eta) (sinkhorn.py:120-136)."""
    kernel = as_device_kernel(kernel)
    torch = _torch()
    with torch.cuda.device(kernel.device):
        sw = _Sweeper(kernel)
        phi, psi = sw.vec(pot.phi), sw.vec(pot.psi)
        rt, ct = sw.vec(as_weights(r)), sw.vec(as_weights(c))   # keep alive until the kernel ran
        lrow, out = sw.vec(), torch.zeros(1, dtype=torch.float64, device=kernel.device)
        sw.row_lse(psi, pot.eta, lrow)
        _lib.check(_lib.lib().leanot_eot_dual(phi.data_ptr(), psi.data_ptr(), rt.data_ptr(), ct.data_ptr(),
                                              lrow.data_ptr(), float(pot.eta), sw.n, out.data_ptr(),
                                              _lib.stream_handle()), "eot_dual")
        return float(out.item())


def sinkhorn_column_marginal(pot: DualPotentials, kernel, workers: int = 1) -> np.ndarray:
    """Column sums of the normalized plan (sinkhorn.py:139-150)."""
    kernel = as_device_kernel(kernel)
    torch = _torch()
    with torch.cuda.device(kernel.device):
        sw = _Sweeper(kernel)
        phi, psi, lcol, col = sw.vec(pot.phi), sw.vec(pot.psi), sw.vec(), sw.vec()
        sw.col_lse(phi, pot.eta, lcol)
        _lib.check(_lib.lib().leanot_sinkhorn_colmarg(psi.data_ptr(), lcol.data_ptr(), float(pot.eta), sw.n,
                                                      col.data_ptr(), _lib.stream_handle()), "colmarg")
        return col.cpu().numpy()


def _potential_plan(kernel, phi, psi, eta: float):
    """exp((phi_i + psi_j - C_ij) / eta) as a device n x n tensor, by the implicit-plan kernel
    (leanot_materialize_plan: r_i exp(-(a C_ij + b_j) - L_i) with a = 1/eta, b = -psi/eta,
    r = 1, L = -phi/eta): the cost is evaluated on device, no dense host copy of C."""
    torch = _torch()
    dev = kernel.device
    n = kernel.n
    with torch.cuda.device(dev):
        b = torch.as_tensor(-np.asarray(psi, dtype=float) / eta, device=dev)
        L = torch.as_tensor(-np.asarray(phi, dtype=float) / eta, device=dev)
        ones = torch.ones(n, dtype=torch.float64, device=dev)
        P = torch.empty((n, n), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().leanot_materialize_plan(kernel.cost_struct(), 1.0 / eta, b.data_ptr(), ones.data_ptr(),
                                                      L.data_ptr(), P.data_ptr(), n, _lib.stream_handle()),
                   "materialize_plan")
    return P


def sinkhorn_plan_dense(pot: DualPotentials, kernel, cap: int = DENSE_CAP) -> np.ndarray:
    """Normalized dense plan, n <= cap (sinkhorn.py:153-159)."""
    kernel = as_device_kernel(kernel)
    if kernel.n > cap:
        raise ValueError("plan materialization above the dense cap")
    plan = _potential_plan(kernel, pot.phi, pot.psi, pot.eta).cpu().numpy()
    return plan / plan.sum()


def ibp_barycenter(kernel, marginals, weights, eta: float, tol: float = 1e-9, max_iter: int = 10_000,
                   workers: int = 1) -> IbpResult:
    """Fixed-support entropic barycenter by iterative Bregman projections (sinkhorn.py:174-228)."""
    if eta <= 0:
        raise ValueError("ibp requires eta > 0")
    m = len(marginals)
    if m == 0:
        raise ValueError("need at least one marginal")
    w = np.asarray(weights, dtype=float).ravel()
    if w.size != m or np.any(w <= 0):
        raise ValueError("weights must be positive, one per marginal")
    w = w / w.sum()
    n = kernel.n
    Ms = [as_weights(h) for h in marginals]
    for ck in Ms:
        if ck.size != n:
            raise ValueError("marginal length mismatch")
        if not bool(np.all(ck > 0)):
            raise ValueError("ibp requires full-support marginals")
    kernel = as_device_kernel(kernel)
    torch = _torch()
    L = _lib.lib()
    dev = kernel.device
    with torch.cuda.device(dev):
        sw = _Sweeper(kernel, batch=m)
        cts = [sw.vec(ck) for ck in Ms]
        phis = torch.zeros((m, n), dtype=torch.float64, device=dev)
        psis = torch.zeros((m, n), dtype=torch.float64, device=dev)
        psis_new = torch.zeros((m, n), dtype=torch.float64, device=dev)
        RL = torch.zeros((m, n), dtype=torch.float64, device=dev)
        log_r = torch.full((n,), -float(np.log(n)), dtype=torch.float64, device=dev)
        wt = sw.vec(w)
        LC = torch.zeros((m, n), dtype=torch.float64, device=dev)
        gaps_t = torch.zeros(m, dtype=torch.float64, device=dev)
        s = _lib.stream_handle()
        gap, converged, sweeps = np.inf, False, 0
        for sweeps in range(1, max_iter + 1):
            sw.col_lse_all(phis, eta, LC)
            for k in range(m):
                _lib.check(L.leanot_sinkhorn_psi(cts[k].data_ptr(), LC[k].data_ptr(), psis[k].data_ptr(), float(eta),
                                                 n, psis_new[k].data_ptr(), gaps_t[k:].data_ptr(), s), "psi")
            gap = float(gaps_t.max().item())
            if sweeps > 1 and gap <= tol:
                converged = True
                break
            psis, psis_new = psis_new, psis
            sw.row_lse_all(psis, eta, RL)
            _lib.check(L.leanot_ibp_rows(wt.data_ptr(), m, n, float(eta), RL.data_ptr(), phis.data_ptr(),
                                         log_r.data_ptr(), s), "ibp_rows")
        lr = log_r.cpu().numpy()
        bary = Histogram.normalized(np.exp(lr - lr.max()))
        return IbpResult(bary, phis.cpu().numpy(), psis.cpu().numpy(), eta, converged, sweeps, gap, log_r=lr)


def ibp_plan_dense(res: IbpResult, kernel, k: int, cap: int = DENSE_CAP) -> np.ndarray:
    """Plan k of an IBP state (sinkhorn.py:231-236)."""
    kernel = as_device_kernel(kernel)
    if kernel.n > cap:
        raise ValueError("plan materialization above the dense cap")
    return _potential_plan(kernel, res.phis[k], res.psis[k], res.eta).cpu().numpy()
