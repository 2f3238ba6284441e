"""B200-native DXG optimal-transport hot path (arXiv 2511.11359), drop-in for `leanot`.

Modules mirror the reference package: `core` (Histogram, cost kernels),
`dxg` (solver), `barycenter`, `rounding`, `sinkhorn` (DualPotentials type).
The n^2 work runs in libleanot_b200.so (hand-written sm_100a CUDA, C ABI in
include/leanot_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
