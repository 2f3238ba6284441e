"""pdxg_reference_step (dxg.py:494-521, the reference's dense equivalence oracle) on the device
kernels leanot_pdxg_rows / leanot_pdxg_colsum (needs a B200).

Pinned to the reference's own 500-iteration dense iterates (tests/golden/spec_acceptance.npz,
written by oracle/gen_golden_spec.py with leanot.dxg.pdxg_reference_step) and to the oracle's
restatement (oracle/leanot_oracle.py:pdxg_step) at a larger n.  Tolerance: 1e-10 absolute on
log_p and delta after 500 steps (north_star: 1e-10 per iteration; the reference's NumPy exp and
the device exp differ by an ulp per element)."""

import numpy as np
import pytest

import leanot_oracle as O
from helpers import load

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [4, 8, 16])
def test_pdxg_reference_step_matches_reference_500_iterations(n):
    from paper_2511_11359_b200 import core, dxg
    d = load("spec_acceptance")
    p = [float(v) for v in d[f"pdxg{n}_params"]]
    prm = dxg.DxgParams(*p)
    C, r, c = d[f"pdxg{n}_C"], d[f"pdxg{n}_r"], d[f"pdxg{n}_c"]
    k = core.ExplicitKernel(C)
    rh, ch = core.Histogram(r), core.Histogram(c)
    st = dxg.pdxg_init(n)
    for _ in range(500):
        st = dxg.pdxg_reference_step(st, k, rh, ch, prm)
    assert np.max(np.abs(st.log_p - d[f"pdxg{n}_log_p"])) <= 1e-10
    assert np.max(np.abs(st.mu.delta - d[f"pdxg{n}_delta"])) <= 1e-10


def test_pdxg_reference_step_matches_oracle_at_n300():
    from paper_2511_11359_b200 import core, dxg
    n = 300
    rng = np.random.default_rng(17)
    C = rng.random((n, n))
    r, c = O.normalized_hist(rng.random(n) + 0.1), O.normalized_hist(rng.random(n) + 0.1)
    k = core.ExplicitKernel(C)
    prm = dxg.params_loose(n, 1e-2, float(c.min()), k.sup_norm)
    oprm = O.Params(prm.eta, prm.eta_mu, prm.tau_p, prm.tau_mu, prm.beta, prm.alpha)
    st = dxg.pdxg_init(n)
    delta, log_p = np.zeros(n), np.full((n, n), -np.log(n))
    Cn = C / C.max()
    for _ in range(5):
        st = dxg.pdxg_reference_step(st, k, core.Histogram(r), core.Histogram(c), prm)
        delta, log_p = O.pdxg_step(delta, log_p, Cn, r, c, oprm, k.sup_norm)
    assert np.max(np.abs(st.log_p - log_p)) <= 1e-12
    assert np.max(np.abs(st.mu.delta - delta)) <= 1e-12


def test_pdxg_reference_step_rejects_size_mismatch():
    from paper_2511_11359_b200 import core, dxg
    k = core.ExplicitKernel(np.random.default_rng(0).random((8, 8)))
    h = core.Histogram(np.full(8, 1 / 8))
    with pytest.raises(ValueError):
        dxg.pdxg_reference_step(dxg.pdxg_init(4), k, h, h, dxg.params_tuned(0.0))
