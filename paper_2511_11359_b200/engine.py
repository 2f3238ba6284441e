"""Device engine of the DXG solver: buffers in HBM, launches through the C ABI.

One `DxgEngine` owns the O(n) state of one solve (dual log-odds delta, plan
log-weights b, scalars a/s/t on device) plus the sweep workspaces, and runs:

    sweep   both column marginals of the current state (pass A + pass B)
            [+ NCCL combine of the column partials when rows are sharded]
    update  the fused O(n) updates of dxg_step (dxg.py:273-278)
    eval    the _evaluate scalars (dxg.py:412-417) from the last eval sweep

Rows can be sharded over a torch.distributed group (one process per GPU):
each rank sweeps rows [row0, row1) of C; the only exchange per iteration is the
2n-vector of column partials (all-gather, summed in rank order so the result is
deterministic), plus 3 scalars on evaluation iterations.
"""

from __future__ import annotations

import os

import ctypes as C

import numpy as np

from . import _lib


def _torch():
    import torch
    return torch


# NVTX ranges around the engine phases (sweep / update / evaluate / iterate) for nsys-style
# timelines: LEANOT_NVTX=1 (off by default: a range push/pop per launch costs a few us)
_NVTX = os.environ.get("LEANOT_NVTX", "0") == "1"


class _nvtx:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if _NVTX:
            _torch().cuda.nvtx.range_push(self.name)

    def __exit__(self, *a):
        if _NVTX:
            _torch().cuda.nvtx.range_pop()


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of rank `rank` (ceil split; trailing ranks may be shorter)."""
    per = (n + world - 1) // world
    return min(n, rank * per), min(n, (rank + 1) * per)


def _host_staged(group) -> bool:
    """Non-NCCL backends (gloo: the CPU tests and multi-process runs on one GPU) exchange
    device tensors through host memory."""
    import torch.distributed as dist
    return dist.get_backend(group) != "nccl"


def all_gather_flat(t, group, world: int):
    """all_gather_into_tensor of a flat copy of `t` (world x numel, rank order), on the
    tensor's device; CUDA tensors are staged through the host on non-NCCL backends."""
    torch = _torch()
    import torch.distributed as dist
    flat = t.contiguous().view(-1)
    if flat.is_cuda and _host_staged(group):
        h = flat.cpu()
        out = torch.empty(world * h.numel(), dtype=h.dtype)
        dist.all_gather_into_tensor(out, h, group=group)
        return out.to(flat.device)
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    return out


def all_reduce_max(t, group):
    """Element-wise MAX over ranks (order-independent, so exact); device tensors are staged
    through the host on non-NCCL backends."""
    import torch.distributed as dist
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        return h.to(t.device)
    out = t.clone()
    dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
    return out


def any_rank(flag: bool, group) -> bool:
    """True on every rank if `flag` is true on any rank (a MAX all-reduce of one int).

    Control decisions taken from per-rank state -- the wall-clock timeout of solve() --
    must agree across ranks, otherwise ranks issue different collectives and hang."""
    if group is None:
        return bool(flag)
    torch = _torch()
    import torch.distributed as dist
    dev = torch.device("cpu") if _host_staged(group) else torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item())


def combine_partials(local, group, world: int):
    """Sum per-rank partial vectors in rank order (all-gather, then fixed-order add).

    Deterministic and identical on every rank regardless of the collective's
    internal reduction order; works for any torch.distributed backend (NCCL on
    the GPU box; gloo with host staging for device tensors, and plain CPU tensors in
    the host-logic tests).
    """
    torch = _torch()
    flat = local.contiguous().view(-1)
    gathered = all_gather_flat(flat, group, world)
    if gathered.is_cuda:
        # rank-order sum on the device (leanot_sum_partials)
        out = torch.empty_like(flat)
        with torch.cuda.device(gathered.device):
            _lib.check(_lib.lib().leanot_sum_partials(gathered.data_ptr(), int(world), flat.numel(), out.data_ptr(),
                                                      _lib.stream_handle()), "sum_partials")
        return out.view(local.shape)
    # CPU tensors: the gloo host-logic tests (tests/test_distributed_gloo.py) only
    gathered = gathered.view((world,) + tuple(local.shape))
    acc = gathered[0].clone()
    for q in range(1, world):
        acc += gathered[q]
    return acc


class DxgEngine:
    def __init__(self, kernel, r, c, params, group=None, device=None, splits=None):
        torch = _torch()
        self.kernel = kernel
        self.device = kernel.device if device is None else torch.device(device)
        self.n = n = kernel.n
        self.group = group
        self.world = 1
        self.rank = 0
        if group is not None:
            import torch.distributed as dist
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        r0, r1 = kernel.local_rows
        if self.world > 1 and kernel.cost_struct().kind == _lib.COST_GRID and (r0, r1) == (0, n):
            # grid costs: separable O(n^1.5) sweeps, replicated on every rank (see BaryEngine)
            self.world, self.rank = 1, 0
        if self.world > 1 and (r0, r1) == (0, n):
            r0, r1 = shard_rows(n, self.world, self.rank)
        if r1 <= r0:
            raise ValueError("empty row shard")
        self.row0, self.row1 = r0, r1
        nr = r1 - r0
        L = _lib.lib()
        if splits is None:
            s = C.c_int(1)
            L.leanot_dxg_default_splits(n, nr, C.byref(s))
            splits = s.value
        nblk = int(min(max(1, (n + 255) // 256), 2 * self._sms()))
        dev = self.device
        f64 = dict(dtype=torch.float64, device=dev)
        rw = np.asarray(r, dtype=float)
        cw = np.asarray(c, dtype=float)
        self.r = torch.from_numpy(rw).to(dev)
        self.c = torch.from_numpy(cw).to(dev)
        self.c_tilde = self.c + params.alpha / n  # c.weights + alpha/n (dxg.py:269)
        self.delta = torch.zeros(n, **f64)
        self.b = torch.zeros(n, **f64)
        self.b_bar = torch.zeros(n, **f64)
        self.bprime = torch.zeros(n, **f64)
        self.sd = torch.zeros(n, **f64)
        self.scal = torch.zeros(8, **f64)
        self.shift = torch.zeros(nr, dtype=torch.int64, device=dev)
        self.m = torch.zeros(2 * nr, dtype=torch.int64, device=dev)
        self.S = torch.zeros(2 * nr, **f64)
        self.coef = torch.zeros(8 * nr, **f64)
        self.rowstat = torch.zeros(3 * nr, **f64)
        if n <= 1024:   # row-owner persistent kernel (csrc/leanot_persist.cu): one partial per CTA
            splits = max(int(splits), self._sms() + 1)
        slab = splits * 2 * n
        if kernel.cost_struct().kind == _lib.COST_GRID:   # separable path scratch (leanot_sep.cu)
            slab = max(slab, int(L.leanot_grid_sep_ws_doubles(kernel.cost_struct())))
        self.slab = torch.zeros(slab, **f64)
        self.col = torch.zeros(2 * n, **f64)
        self.partial = torch.zeros(2 * nblk, **f64)
        self.evalbuf = torch.zeros(16, **f64)
        self.flags = torch.zeros(2 + 4 * nr, dtype=torch.int32, device=dev)
        # expanded-form sweeps of squared-Euclidean points (leanot_cost_t.norms): beta_0 | beta_1,
        # each padded to an even length
        self.beta = torch.zeros(2 * (n + 1), **f64) if kernel.cost_struct().norms else None
        self.params = params
        self.plan = _lib.DxgPlanT()
        p = self.plan
        p.cost = kernel.cost_struct()
        p.prm = _lib.ParamsT(params.eta, params.eta_mu, params.tau_p, params.tau_mu, params.beta, params.alpha)
        p.n, p.row0, p.row1, p.splits, p.nblk_upd = n, r0, r1, int(splits), nblk
        for name in ("r", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "m", "S",
                     "coef", "rowstat", "slab", "col", "partial", "evalbuf", "flags"):
            setattr(p, name, getattr(self, name).data_ptr())
        p.beta = self.beta.data_ptr() if self.beta is not None else None
        self._graphs = {}
        self._h_in = self._h_out = None
        pos = rw > 0
        self.h_r = float(-(rw[pos] * np.log(rw[pos])).sum())  # H(r) (dxg.py:308-309, 340-341)

    def _sms(self):
        v = C.c_int(148)
        _lib.lib().leanot_device_sm_count(self.device.index or 0, C.byref(v))
        return v.value

    # -- state ------------------------------------------------------------------
    def load_state(self, delta, b, a, s, t, fresh=False, keep_shift=False):
        """Upload a state (H2D) and derive the midpoint weights.  fresh: the zero state of
        solve(); keep_shift: the state this engine produced last (warm row shifts);
        otherwise row maxima are computed (injected state)."""
        torch = _torch()
        n = self.delta.numel()
        if self._h_in is None:   # pinned staging: true async H2D, no pageable bounce
            self._h_in = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
            self._h_out = torch.empty(2 * n + 4, dtype=torch.float64, pin_memory=True)
            self._h_in_done = torch.cuda.Event()
        else:
            self._h_in_done.synchronize()   # the previous upload has left the staging buffer
        hv = self._h_in.numpy()
        hv[:n] = np.asarray(delta, dtype=float)
        hv[n:] = np.asarray(b, dtype=float)
        with torch.cuda.device(self.device):
            self.delta.copy_(self._h_in[:n], non_blocking=True)
            self.b.copy_(self._h_in[n:], non_blocking=True)
            self._h_in_done.record()
        mode = 1 if fresh else (2 if keep_shift else 0)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().leanot_dxg_prepare(C.byref(self.plan), float(a), float(s), float(t),
                                                     mode, _lib.stream_handle()), "dxg_prepare")

    def read_state(self):
        torch = _torch()
        if self._h_out is None:
            sc = self.scal[:4].cpu().tolist()
            return self.delta.cpu().numpy(), self.b.cpu().numpy(), sc[0], sc[2], int(round(sc[3]))
        n = self.delta.numel()
        with torch.cuda.device(self.device):   # one sync for delta, b and the scalars
            self._h_out[:n].copy_(self.delta, non_blocking=True)
            self._h_out[n:2 * n].copy_(self.b, non_blocking=True)
            self._h_out[2 * n:].copy_(self.scal[:4], non_blocking=True)
            torch.cuda.current_stream().synchronize()
        ho = self._h_out.numpy()
        sc = ho[2 * n:].tolist()
        return ho[:n].copy(), ho[n:2 * n].copy(), sc[0], sc[2], int(round(sc[3]))

    def scalars(self):
        return self.scal[:4].cpu().tolist()

    # -- iteration ---------------------------------------------------------------
    def _stream(self):
        return _lib.stream_handle()

    def sweep(self, evaluate=False, fused=False, single_read=None):
        """fused: stored costs only -- the experimental L2-reuse sweep (csrc/leanot_fused.cu).
        single_read: None = library default (the single-read, single-exp sweep of
        csrc/leanot_sr.cu for stored costs with n >= 32768), True = force it (any eligible n),
        False = the two-pass sweep."""
        flags = (1 if evaluate else 0) | (8 if fused else 0)
        if single_read is True:
            flags |= 32
        elif single_read is False:
            flags |= 16
        with _nvtx("leanot.sweep.eval" if evaluate else "leanot.sweep"), _torch().cuda.device(self.device):
            _lib.check(_lib.lib().leanot_dxg_sweep(C.byref(self.plan), flags, self._stream()), "dxg_sweep")
        if self.world > 1:
            self._combine_cols()

    def sweep_phase(self, phase: str):
        """Run only pass A ("rows") or only pass B ("cols") -- for per-kernel timing."""
        flag = {"rows": 2, "cols": 4}[phase]
        with _torch().cuda.device(self.device):
            _lib.check(_lib.lib().leanot_dxg_sweep(C.byref(self.plan), flag, self._stream()), "dxg_sweep")
        if phase == "cols" and self.world > 1:
            self._combine_cols()

    def _combine_cols(self):
        self.col.copy_(combine_partials(self.col, self.group, self.world))

    def update(self):
        with _nvtx("leanot.update"), _torch().cuda.device(self.device):
            _lib.check(_lib.lib().leanot_dxg_update(C.byref(self.plan), self._stream()), "dxg_update")

    def iterate(self, iters: int, use_graph: bool | None = None):
        """iters x (sweep, update) with no evaluation."""
        if iters <= 0:
            return
        if self.world > 1:
            for _ in range(iters):
                self.sweep()
                self.update()
            return
        L = _lib.lib()
        if use_graph is None:
            # n <= 4096: leanot_dxg_iterate runs all iterations in one persistent kernel
            persistent = self.n <= 4096 and os.environ.get("LEANOT_PERSIST", "1") != "0"
            use_graph = self.n <= 20000 and not persistent
        with _torch().cuda.device(self.device):
            if not use_graph:
                _lib.check(L.leanot_dxg_iterate(C.byref(self.plan), int(iters), self._stream()), "dxg_iterate")
                return
            g = self._graphs.get(iters)
            if g is None:
                h = C.c_void_p()
                _lib.check(L.leanot_graph_create(C.byref(self.plan), int(iters), C.byref(h), self._stream()),
                           "graph_create")
                g = self._graphs[iters] = h
            _lib.check(L.leanot_graph_launch(g, self._stream()), "graph_launch")

    def evaluate(self):
        """(primal, dual, infeas, s) of the state swept by the last sweep(evaluate=True)."""
        torch = _torch()
        with _nvtx("leanot.eval"), torch.cuda.device(self.device):
            _lib.check(_lib.lib().leanot_dxg_eval(C.byref(self.plan), self._stream()), "dxg_eval")
        # the scalars (a, a_bar, s, t) travel in the same device->host transfer
        self.evalbuf[8:12].copy_(self.scal[:4])
        return self.evaluate_buffer()

    def evaluate_buffer(self):
        """(primal, dual, infeas) from evalbuf[0..4] (+ scalars in [8..11]) as filled by
        leanot_dxg_eval or leanot_dxg_iterate_eval."""
        buf = self.evalbuf[:5]
        if self.world > 1:
            cost_v, ent_rows, inner_rows = combine_partials(buf[:3], self.group, self.world).cpu().tolist()
            tail = self.evalbuf[3:12].cpu().tolist()
            infeas, cd = tail[0], tail[1]
            self.last_scalars = tail[5:9]
        else:
            vals = self.evalbuf[:12].cpu().tolist()
            cost_v, ent_rows, inner_rows, infeas, cd = vals[:5]
            self.last_scalars = vals[8:12]
        eta = self.params.eta
        sup = self.kernel.sup_norm
        ent = ent_rows + self.h_r
        primal = cost_v + 2.0 * sup * infeas - eta * ent            # dxg.py:415
        if eta > 0:
            inner = -eta * inner_rows - eta * self.h_r                # dxg.py:342
        else:
            inner = inner_rows                                       # dxg.py:348
        dual = float(-2.0 * sup * cd + inner)                        # dxg.py:349
        return primal, dual, infeas

    def col_now(self):
        return self.col[: self.n].cpu().numpy()

    def close(self):
        L = _lib.lib()
        for g in self._graphs.values():
            L.leanot_graph_destroy(g)
        self._graphs.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_group():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return dist.group.WORLD
    except Exception:
        pass
    return None

