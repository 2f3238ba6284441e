"""The η > 0 evaluation row LSE takes its shift from pass A's row minima
(csrc/leanot_solver.cu leanot_dxg_eval, csrc/leanot_bary.cu leanot_bary_eval):
max_j fl(x_j * s) == fl(min_j x_j * s) for s < 0, because IEEE round-to-nearest
multiplication is monotone.  Checked here on adversarial FP64 data (near-ties,
subnormal-adjacent and large magnitudes) so the "exact shift" claim is pinned on CPU.
"""
import numpy as np
import pytest


@pytest.mark.parametrize("seed", range(8))
def test_max_of_scaled_equals_scaled_min(seed):
    rng = np.random.default_rng(seed)
    for _ in range(200):
        n = int(rng.integers(1, 400))
        base = rng.normal(scale=10.0 ** rng.integers(-300, 300))
        # near-ties: values one or two ulps apart around a common base
        x = base + np.spacing(base) * rng.integers(-3, 4, size=n)
        x = np.concatenate([x, rng.normal(size=n) * 10.0 ** rng.integers(-5, 5)])
        s = -1.0 / float(10.0 ** rng.uniform(-4, 3))
        assert np.max(x * s) == np.min(x) * s


def test_table_exp_argument_never_positive_with_exact_shift():
    rng = np.random.default_rng(1)
    C = rng.random((64, 257))
    sd = rng.normal(size=257)
    eta = 1e-3
    x = C + sd
    xm = x.min(axis=1) * (-1.0 / eta)
    y = x * (-1.0 / eta) - xm[:, None]
    assert (y <= 0).all() and (y.max(axis=1) == 0).all()
