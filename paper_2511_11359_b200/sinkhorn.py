"""Dual potentials type shared with the DXG potential recovery (sinkhorn.py:30-44).

The Sinkhorn/IBP baselines themselves are outside the hot-path scope of this
round; only the result type returned by
dxg.recover_eot_potentials lives here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["DualPotentials"]


@dataclass
class DualPotentials:
    phi: np.ndarray
    psi: np.ndarray
    eta: float
    converged: bool = True
    sweeps: int = 0
    col_gap: float = field(default=np.nan)
