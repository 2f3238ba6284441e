"""Out-of-bounds writes and races without compute-sanitizer (needs a B200).

compute-sanitizer is closed on the GPU pool this project runs on, so the same classes of bug
are checked with the tools the kernels allow:

* guard bands: every device buffer of a plan (state, row outputs, slabs, scratch, flags) is
  moved into the middle of a larger allocation whose head and tail hold a sentinel bit
  pattern; after sweeps, updates and evaluations of every kernel family the sentinels must
  be intact (an out-of-bounds store anywhere near a buffer changes them);
* determinism: the same sweep from the same state, repeated, must give bitwise identical
  outputs (a shared-memory or cross-CTA race in a reduction shows up as run-to-run
  differences; the reductions are fixed-order by design, core.py:297-309).

Kernel families: TMA two-pass (stored C), on-the-fly points (expanded and difference form),
persistent iterate (1024 < n <= 4096), row-owner (n <= 1024), L2-reuse fused sweep,
single-read sweep, separable grid (DXG + barycenter), dense barycenter.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PAD = 2048
SENTINEL = 0x7FF4_DEAD_BEEF_0BAD   # a NaN payload no kernel writes


def _guard(eng, names):
    """Move eng.<name> into the middle of a guarded allocation; returns the checker."""
    import torch
    guards = []
    for name in names:
        t = getattr(eng, name, None)
        if t is None:
            continue
        nbytes = t.numel() * t.element_size()
        words = (nbytes + 7) // 8
        big = torch.empty(2 * PAD + words, dtype=torch.int64, device=t.device)
        big[:PAD] = SENTINEL
        big[PAD + words:] = SENTINEL
        mid = big[PAD:PAD + words].view(torch.uint8)[:nbytes].view(t.dtype)
        mid.copy_(t.view(-1))
        new = mid.view(t.shape)
        setattr(eng, name, new)
        setattr(eng.plan, name, new.data_ptr())
        guards.append((name, big, words))

    def check():
        torch.cuda.synchronize()
        for name, big, words in guards:
            head = big[:PAD]
            tail = big[PAD + words:]
            assert bool((head == head[0]).all()) and bool((tail == head[0]).all()), f"guard band of {name} overwritten"
    return check


DXG_BUFS = ("r", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "m", "S", "coef", "rowstat",
            "slab", "col", "partial", "evalbuf", "flags", "beta")
BARY_BUFS = ("w", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "mu", "S", "L", "r", "coef",
             "rowstat", "slab", "col", "partial", "scratch", "evalbuf", "flags")


def _hist(rng, n):
    w = rng.random(n) + 0.05
    return w / w.sum()


def _dxg_case(case):
    from paper_2511_11359_b200 import core
    import zlib
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    if case == "tma":
        k = core.HashKernel(4096, seed=1)
    elif case == "tma_shard":
        k = core.HashKernel(6000, seed=1, rows=(1001, 4003))
    elif case == "gram":
        k = core.ColorKernel(rng.random((3001, 3)) + 5.0, 2)
    elif case == "diff":
        k = core.ColorKernel(rng.random((3001, 3)), 2)
        k.norms_dev = None
    elif case in ("persist", "persist_graph"):
        k = core.HashKernel(2500, seed=2)
    elif case == "rowowner":
        k = core.ExplicitKernel(rng.random((700, 700)))
    elif case == "fused":
        k = core.HashKernel(16384, seed=3)
    elif case == "sr":
        k = core.HashKernel(3000, seed=4)
    elif case == "grid":
        k = core.GridKernel(20, 18, 2)
    return k, rng


@pytest.mark.parametrize("case", ["tma", "tma_shard", "gram", "diff", "persist", "rowowner", "fused", "sr", "grid"])
def test_dxg_kernels_respect_buffer_bounds_and_are_deterministic(case):
    import torch
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200.engine import DxgEngine
    k, rng = _dxg_case(case)
    n = k.n
    prm = dxg.params_tuned(1e-3).with_overrides(tau_mu=0.05)
    eng = DxgEngine(k, _hist(rng, n), _hist(rng, n), prm)
    check = _guard(eng, DXG_BUFS)
    b = -np.abs(rng.normal(0, 2.0, n))
    st = (rng.uniform(-1, 1, n), b - b.max(), 40.0, 0.1, 40)
    fused = case == "fused"
    sr = True if case == "sr" else None
    outs = []
    for rep in range(2):
        eng.load_state(*st)
        for _ in range(3):
            eng.sweep(fused=fused, single_read=sr)
            eng.update()
        if case in ("persist", "rowowner"):
            eng.iterate(7, use_graph=False)       # the persistent kernels (n <= 4096)
        eng.sweep(evaluate=True)
        ev = eng.evaluate()
        eng.scal[0] = 3000.0                      # forced fixup rows (exact recompute path)
        eng.sweep(fused=fused, single_read=sr)
        torch.cuda.synchronize()
        outs.append([x.clone() for x in (eng.col, eng.S, eng.m, eng.shift, eng.delta, eng.b)] + [ev])
        check()
    for x, y in zip(outs[0][:-1], outs[1][:-1]):
        assert torch.equal(x, y)
    assert outs[0][-1] == outs[1][-1]


def test_rowowner_iterate_eval_respects_bounds():
    from paper_2511_11359_b200 import dxg
    from paper_2511_11359_b200 import _lib
    import ctypes as C
    import torch
    from paper_2511_11359_b200.engine import DxgEngine
    k, rng = _dxg_case("rowowner")
    n = k.n
    eng = DxgEngine(k, _hist(rng, n), _hist(rng, n), dxg.params_tuned(0.0).with_overrides(tau_mu=0.05))
    check = _guard(eng, DXG_BUFS)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    res = []
    for _ in range(2):
        _lib.check(_lib.lib().leanot_dxg_iterate_eval(C.byref(eng.plan), 25, 0, _lib.stream_handle()), "iterate_eval")
        res.append(eng.evaluate_buffer())
    torch.cuda.synchronize()
    check()


@pytest.mark.parametrize("kind", ["grid", "points"])
def test_barycenter_kernels_respect_buffer_bounds_and_are_deterministic(kind):
    import torch
    from paper_2511_11359_b200 import barycenter as B
    from paper_2511_11359_b200 import core, dxg
    rng = np.random.default_rng(9)
    g = core.GridKernel(14, 16, 2) if kind == "grid" else core.ColorKernel(rng.random((500, 2)), 2)
    n, m = g.n, 3
    margs = [core.Histogram(_hist(rng, n)) for _ in range(m)]
    prm = dxg.params_tuned(1e-2).with_overrides(tau_mu=0.05)
    eng = B.BaryEngine(g, margs, np.array([0.2, 0.5, 0.3]), prm)
    check = _guard(eng, BARY_BUFS)
    deltas = rng.uniform(-0.5, 0.5, (m, n))
    bs = -np.abs(rng.normal(0, 1.0, (m, n)))
    outs = []
    for _ in range(2):
        eng.load_state(deltas, bs, 9.0, 0.01, 9)
        for _ in range(4):
            eng.sweep()
            eng.update()
        eng.sweep(evaluate=True)
        p, d, inf = eng.evaluate()
        torch.cuda.synchronize()
        outs.append([eng.col.clone(), eng.r.clone(), eng.L.clone(), eng.delta.clone(), (p, d, tuple(inf))])
        check()
    for x, y in zip(outs[0][:-1], outs[1][:-1]):
        assert torch.equal(x, y)
    assert outs[0][-1] == outs[1][-1]
