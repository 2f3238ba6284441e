"""Histograms and device-resident cost kernels (drop-in for leanot.core).

Mirrors the reference's CostKernel plugin protocol (core.py:167-192): every
kernel exposes `n`, `scale` (raw sup-norm divided out), `sup_norm` (1, or 0 for
an all-zero matrix), `block(i0, i1)`, `entry(i, j)` and `materialize(cap)`.  The
difference is where the data lives: the kernels hold their cost description in
HBM and hand the CUDA sweeps a `leanot_cost_t` descriptor; `block()` is
evaluated by a device kernel and exists for compatibility (rounding, tests).

Extensions (not in the reference): `ExplicitKernel` accepts a CUDA tensor and
`cap=None` so an 80 GB matrix can live in HBM without a host copy;
`HashKernel` generates the counter-based stored-C benchmark instance on
device; `ColorKernel(..., scale=)` skips the O(n^2 d) sup pass when the scale
is known by construction; any kernel can be restricted to a row range
(`rows=`) for row sharding across GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["DENSE_CAP", "BLOCK_ROWS", "Histogram", "CostKernel", "GridKernel", "ExplicitKernel",
           "ColorKernel", "HashKernel", "cost_eval", "iter_blocks", "map_blocks", "ingest_image_histogram", "lse",
           "lse_rows", "kl_divergence", "entropy", "logistic"]

DENSE_CAP = 4096      # core.py:40
BLOCK_ROWS = 128      # core.py:44 (the GPU sweeps do not use host row blocks)
_SIMPLEX_ATOL = 1e-12  # core.py:46


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class Histogram:
    """Probability mass function on the n-point simplex (core.py:107-144)."""

    weights: np.ndarray
    full_support: bool = field(default=False)

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float).ravel()
        if w.size == 0:
            raise ValueError("empty histogram")
        if np.any(w < 0):
            raise ValueError("histogram entries must be nonnegative")
        if abs(w.sum() - 1.0) > _SIMPLEX_ATOL:
            raise ValueError(f"histogram sums to {w.sum()!r}, not 1")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "full_support", bool(np.all(w > 0)))

    @classmethod
    def normalized(cls, raw) -> "Histogram":
        raw = np.asarray(raw, dtype=float).ravel()
        total = raw.sum()
        if total <= 0:
            raise ValueError("cannot normalize: total mass is not positive")
        return cls(raw / total)

    @property
    def n(self) -> int:
        return self.weights.size

    def min(self) -> float:
        return float(self.weights.min())


def ingest_image_histogram(pixels, perturbation: float = 1e-6) -> Histogram:
    """Grayscale image -> full-support row-major histogram (core.py:147-164).

    Unit-mass normalization, + `perturbation` per pixel, renormalized; with a
    zero perturbation exact zeros are kept (full_support False).  Same checks
    and ValueError messages as the reference.
    """
    img = np.asarray(pixels, dtype=float)
    if np.any(img < 0):
        raise ValueError("image has negative pixels")
    total = img.sum()
    if total <= 0:
        raise ValueError("image has no positive pixel")
    h = img.ravel(order="C") / total
    if perturbation != 0.0:
        h = h + perturbation
        h = h / h.sum()
    return Histogram(h)


# O(n) host helpers of the reference's public core surface (core.py:49-103).  The solvers
# never call them on the n^2 path (their LSEs / entropies run in the CUDA sweeps); they are
# here so user code importing them from leanot.core keeps working.

def lse(values) -> float:
    """Max-shifted log-sum-exp of a 1-D sequence (core.py:49-64); all -inf -> -inf."""
    v = np.asarray(values, dtype=float)
    if v.size == 0:
        raise ValueError("lse of an empty sequence")
    m = v.max()
    if not np.isfinite(m):
        if m == -np.inf:
            return -np.inf
        raise ValueError("lse input contains +inf or NaN")
    return float(m + np.log(np.exp(v - m).sum()))


def lse_rows(z) -> np.ndarray:
    """Row-wise log-sum-exp of a 2-D array (core.py:67-70)."""
    z = np.asarray(z, dtype=float)
    m = z.max(axis=1)
    return m + np.log(np.exp(z - m[:, None]).sum(axis=1))


def kl_divergence(a, b) -> float:
    """<a, log a - log b>, 0 log 0 = 0; a must be absolutely continuous w.r.t. b (core.py:73-86)."""
    a = np.asarray(a, dtype=float).ravel()
    b = np.asarray(b, dtype=float).ravel()
    if a.shape != b.shape:
        raise ValueError("kl_divergence: shape mismatch")
    pos = a > 0
    if np.any(b[pos] <= 0):
        raise ValueError("kl_divergence: a is not absolutely continuous w.r.t. b")
    return float(np.sum(a[pos] * (np.log(a[pos]) - np.log(b[pos]))))


def entropy(weights) -> float:
    """-sum x log x with 0 log 0 = 0 (core.py:89-93)."""
    x = np.asarray(weights, dtype=float).ravel()
    pos = x > 0
    return float(-np.sum(x[pos] * np.log(x[pos])))


def logistic(x) -> np.ndarray:
    """Overflow-free elementwise sigmoid (core.py:96-104)."""
    x = np.asarray(x, dtype=float)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def as_weights(h) -> np.ndarray:
    """Accept a Histogram (ours or the reference's) or an array."""
    return np.asarray(getattr(h, "weights", h), dtype=float).ravel()


class CostKernel:
    """Device-resident normalized nonnegative cost (core.py:167-192)."""

    n: int
    scale: float
    sup_norm: float
    row0: int = 0
    row1: int | None = None

    def __init__(self, device=None):
        torch = _torch()
        _lib.require_cuda()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    # -- descriptor handed to the C ABI -----------------------------------------
    def cost_struct(self) -> _lib.CostT:
        raise NotImplementedError

    @property
    def local_rows(self) -> tuple[int, int]:
        return (self.row0, self.n if self.row1 is None else self.row1)

    # -- reference protocol -------------------------------------------------------
    def block(self, i0: int, i1: int) -> np.ndarray:
        r0, r1 = self.local_rows
        if not (r0 <= i0 <= i1 <= r1):
            raise IndexError("block rows outside the rows held by this kernel")
        torch = _torch()
        out = torch.empty((max(i1 - i0, 0), self.n), dtype=torch.float64, device=self.device)
        if i1 > i0:
            with torch.cuda.device(self.device):
                st = self.cost_struct()
                _lib.check(_lib.lib().leanot_cost_block(st, i0, i1, out.data_ptr(), self.n,
                                                          _lib.stream_handle()), "cost_block")
        return out.cpu().numpy()

    def entry(self, i: int, j: int) -> float:
        if not (0 <= i < self.n and 0 <= j < self.n):
            raise IndexError("cost index out of range")
        return float(self.block(i, i + 1)[0, j])

    def materialize(self, cap: int = DENSE_CAP) -> np.ndarray:
        if self.n > cap:
            raise ValueError(f"refusing to materialize {self.n}x{self.n} cost matrix (cap {cap})")
        return self.block(0, self.n)


def cost_eval(kernel: CostKernel, i: int, j: int) -> float:
    return kernel.entry(i, j)


def iter_blocks(n: int, block_rows: int = BLOCK_ROWS):
    for i0 in range(0, n, block_rows):
        yield i0, min(i0 + block_rows, n)


def map_blocks(fn, n: int, workers: int = 1, block_rows: int = BLOCK_ROWS) -> list:
    """fn(i0, i1) over the row blocks, results in block order (core.py:297-309).

    Kept for user plug-ins that stream `block()`; the CUDA solvers never call it (their
    row blocks are CTAs, reduced in a fixed order on device).  With workers > 1 the
    blocks run on a thread pool but are consumed in block order (deterministic).
    """
    ranges = list(iter_blocks(n, block_rows))
    if workers <= 1 or len(ranges) == 1:
        return [fn(i0, i1) for i0, i1 in ranges]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futures = [pool.submit(fn, i0, i1) for i0, i1 in ranges]
        return [f.result() for f in futures]


def _even(n: int) -> int:
    return n + (n & 1)


class ExplicitKernel(CostKernel):
    """Dense cost normalized on device (core.py:239-261).

    `matrix` may be a host array or a CUDA float64 tensor (no host copy).  The
    normalized copy lives in HBM with an even leading dimension.
    """

    def __init__(self, matrix, cap: int | None = DENSE_CAP, device=None):
        torch = _torch()
        if isinstance(matrix, torch.Tensor) and matrix.is_cuda:
            device = matrix.device if device is None else device
        super().__init__(device)
        if isinstance(matrix, torch.Tensor):
            m = matrix.to(device=self.device, dtype=torch.float64)
        else:
            arr = np.asarray(matrix, dtype=float)
            if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
                raise ValueError("explicit cost matrix must be square")
            m = torch.from_numpy(np.ascontiguousarray(arr))
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("explicit cost matrix must be square")
        n = int(m.shape[0])
        if cap is not None and n > cap:
            raise ValueError(f"explicit kernel of size {n} exceeds dense cap {cap}")
        self.n = n
        self.ld = _even(n)
        self.mat = torch.zeros((n, self.ld), dtype=torch.float64, device=self.device)
        self.mat[:, :n].copy_(m, non_blocking=False)
        del m
        self._normalize()

    def _normalize(self):
        torch = _torch()
        n = self.n
        scratch = torch.empty(2048 + 2, dtype=torch.float64, device=self.device)
        out = scratch[2048:]
        L = _lib.lib()
        with torch.cuda.device(self.device):
            s = _lib.stream_handle()
            _lib.check(L.leanot_stored_max(self.mat.data_ptr(), n, n, self.ld, out.data_ptr(),
                                           scratch.data_ptr(), s), "stored_max")
            mx, neg_min = out.cpu().tolist()
        if -neg_min < 0:
            raise ValueError("cost entries must be nonnegative")
        raw_sup = float(mx)
        self.scale = raw_sup if raw_sup > 0 else 1.0
        self.sup_norm = 1.0 if raw_sup > 0 else 0.0
        with torch.cuda.device(self.device):
            _lib.check(L.leanot_stored_normalize(self.mat.data_ptr(), n, n, self.ld, self.scale,
                                                 _lib.stream_handle()), "stored_normalize")

    def cost_struct(self) -> _lib.CostT:
        return _lib.CostT(kind=_lib.COST_STORED, n=self.n, ld=self.ld, row_base=self.row0,
                          mat=self.mat.data_ptr(), inv_scale=1.0 / self.scale, sup_norm=self.sup_norm)


class HashKernel(CostKernel):
    """Stored-C benchmark instance generated in HBM (BASELINE config 3).

    C_ij = splitmix64(seed, i, j) -> U[0,1) and C[0][n-1] = 1, so the raw
    sup-norm is 1 by construction (scale = 1).  `rows=(r0, r1)` allocates only
    those rows (row sharding).  The host regenerates any block with
    oracle/leanot_oracle.py:HashCost.
    """

    def __init__(self, n: int, seed: int = 0, rows: tuple[int, int] | None = None, device=None):
        super().__init__(device)
        torch = _torch()
        self.n, self.seed = int(n), int(seed)
        self.row0, self.row1 = (0, self.n) if rows is None else (int(rows[0]), int(rows[1]))
        self.ld = _even(self.n)
        nr = self.row1 - self.row0
        self.mat = torch.empty((nr, self.ld), dtype=torch.float64, device=self.device)
        self.scale, self.sup_norm = 1.0, 1.0
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().leanot_hash_fill(self.mat.data_ptr(), self.row0, nr, self.n, self.ld,
                                                   self.seed, _lib.stream_handle()), "hash_fill")
        if self.ld > self.n:
            self.mat[:, self.n:].zero_()

    def cost_struct(self) -> _lib.CostT:
        return _lib.CostT(kind=_lib.COST_STORED, n=self.n, ld=self.ld, row_base=self.row0,
                          mat=self.mat.data_ptr(), inv_scale=1.0, sup_norm=self.sup_norm)


class GridKernel(CostKernel):
    """(|drow|^p + |dcol|^p) / ((H-1)^p + (W-1)^p) on an H x W grid (core.py:200-236)."""

    def __init__(self, height: int, width: int, p: int = 2, device=None):
        if height < 1 or width < 1:
            raise ValueError("grid dimensions must be positive")
        if p not in (1, 2, 3):
            raise ValueError("grid exponent p must be 1, 2 or 3")
        super().__init__(device)
        torch = _torch()
        self.height, self.width, self.p = int(height), int(width), int(p)
        self.n = self.height * self.width
        raw_sup = float((self.height - 1) ** p + (self.width - 1) ** p)
        self.scale = raw_sup if raw_sup > 0 else 1.0
        self.sup_norm = 1.0 if raw_sup > 0 else 0.0
        k = torch.arange(self.n, dtype=torch.int64, device=self.device)
        self.coords = torch.cat([(k // self.width).double(), (k % self.width).double()])

    def cost_struct(self) -> _lib.CostT:
        return _lib.CostT(kind=_lib.COST_GRID, p=self.p, height=self.height, width=self.width, n=self.n,
                          grid_coords=self.coords.data_ptr(), inv_scale=1.0 / self.scale,
                          sup_norm=self.sup_norm)


class ColorKernel(CostKernel):
    """sum_d |f_id - f_jd|^p between n feature vectors (core.py:264-288).

    The sup-norm is exact (one O(n^2 d) device pass, as core.py:279-284) unless
    `scale` is given.  Feature dimension 1..4 (RGB is 3).
    """

    def __init__(self, features, p: int = 2, scale: float | None = None, device=None):
        torch = _torch()
        if isinstance(features, torch.Tensor):
            f = features.detach().to(dtype=torch.float64)
            if f.ndim != 2:
                raise ValueError("features must be an (n, d) array")
        else:
            f = np.asarray(features, dtype=float)
            if f.ndim != 2:
                raise ValueError("features must be an (n, d) array")
            f = torch.from_numpy(np.ascontiguousarray(f))
        if p not in (1, 2, 3):
            raise ValueError("exponent p must be 1, 2 or 3")
        if not (1 <= f.shape[1] <= 4):
            raise ValueError("device ColorKernel supports feature dimension 1..4")
        super().__init__(device)
        self.features_dev = f.to(self.device).contiguous()
        self.p = int(p)
        self.n, self.dim = int(f.shape[0]), int(f.shape[1])
        if scale is None:
            scratch = torch.empty(1025, dtype=torch.float64, device=self.device)
            with torch.cuda.device(self.device):
                _lib.check(_lib.lib().leanot_points_sup(self.features_dev.data_ptr(), self.n, self.dim, self.p,
                                                        scratch[1024:].data_ptr(), scratch.data_ptr(),
                                                        _lib.stream_handle()), "points_sup")
            raw_sup = float(scratch[1024].item())
        else:
            raw_sup = float(scale)
        self.scale = raw_sup if raw_sup > 0 else 1.0
        self.sup_norm = 1.0 if raw_sup > 0 else 0.0
        self.norms_dev = None
        if self.p == 2:  # |f_j|^2 for the expanded-form sweeps (leanot_cost_t.norms)
            # [|f_j - mu|^2 (n, even-padded) | centered features (n x dim) | mu] (leanot_points_norms)
            npad = (self.n + 1) & ~1
            self.norms_dev = torch.empty(npad + self.n * self.dim + self.dim, dtype=torch.float64, device=self.device)
            with torch.cuda.device(self.device):
                _lib.check(_lib.lib().leanot_points_norms(self.features_dev.data_ptr(), self.n, self.dim,
                                                          self.norms_dev.data_ptr(), _lib.stream_handle()),
                           "points_norms")

    @property
    def features(self) -> np.ndarray:
        return self.features_dev.cpu().numpy()

    def cost_struct(self) -> _lib.CostT:
        return _lib.CostT(kind=_lib.COST_POINTS, p=self.p, dim=self.dim, n=self.n,
                          feat=self.features_dev.data_ptr(), inv_scale=1.0 / self.scale,
                          sup_norm=self.sup_norm,
                          norms=self.norms_dev.data_ptr() if self.norms_dev is not None else None)


def as_device_kernel(kernel, device=None) -> CostKernel:
    """Wrap a reference CostKernel (leanot.core) into the device equivalent.

    Lets users hand the reference's kernel objects to this package unchanged.
    """
    if isinstance(kernel, CostKernel):
        return kernel
    name = type(kernel).__name__
    if name == "GridKernel":
        return GridKernel(kernel.height, kernel.width, kernel.p, device=device)
    if name == "ColorKernel":
        return ColorKernel(kernel.features, kernel.p, scale=kernel.scale if kernel.sup_norm else 0.0, device=device)
    if name == "ExplicitKernel" or hasattr(kernel, "materialize"):
        m = kernel.materialize(kernel.n)
        k = ExplicitKernel(m, cap=None, device=device)
        # the reference kernel already normalized; keep its scale for reporting
        k.scale, k.sup_norm = kernel.scale, kernel.sup_norm
        return k
    raise TypeError(f"unsupported cost kernel {name}")
