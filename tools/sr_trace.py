"""Per-panel timestamps of the single-read sweep (debug trace, csrc/leanot_sr.cu).

    python tools/sr_trace.py [--n 100000] [--rows 16000]

Sweeps a row shard [0, rows) of the n = 1e5 hash matrix (npan = rows / 4 <= 4096 panels)
and prints, for CTAs 0 and G-1: the panel period, publish->summed latency and
summed->posted time (us).
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import torch  # noqa: E402

from paper_2511_11359_b200 import _lib, core, dxg  # noqa: E402
from paper_2511_11359_b200.engine import DxgEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--rows", type=int, default=16000)
a = ap.parse_args()
n = a.n
rng = np.random.default_rng(1)
r, c = rng.random(n), rng.random(n)
k = core.HashKernel(n, seed=0, rows=(0, a.rows))
prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
eng = DxgEngine(k, r / r.sum(), c / c.sum(), prm)
eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
for _ in range(3):
    eng.sweep(single_read=True)
    eng.update()
tr = torch.zeros(2 * 8 * 4096, dtype=torch.int64, device="cuda")
_lib.lib().leanot_debug_sr_trace(tr.data_ptr())
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
eng.sweep(single_read=True)
e1.record(st)
torch.cuda.synchronize()
_lib.lib().leanot_debug_sr_trace(None)
ms = e0.elapsed_time(e1)
npan = (a.rows + 3) // 4
print(f"sweep {ms:.3f} ms for {a.rows} rows ({npan} panels): {ms * 1e3 / npan:.3f} us/panel")
t = tr.cpu().numpy().reshape(2, 4096, 8)[:, :npan, :].astype(np.float64)
names = ["pub", "coll_start", "buf_ready", "polled", "posted", "cons_wait", "cons_got", "rounds"]
for nm, x in (("cta0", t[0]), ("ctaG-1", t[1])):
    sl = slice(npan // 4, 3 * npan // 4)
    cyc_per_us = (x[3 * npan // 4, 0] - x[npan // 4, 0]) / (ms * 1e3 / npan * (npan // 2))
    print(f"{nm}: clock {cyc_per_us:.0f} cyc/us; per-panel medians in cycles:")
    d = lambda i, j, off=0: np.median(x[sl, i][off:] - x[sl, j][:len(x[sl, j]) - off] if off else x[sl, i] - x[sl, j])
    print(f"  period(pub) {np.median(np.diff(x[sl, 0])):.0f}  period(posted) {np.median(np.diff(x[sl, 4])):.0f}")
    print(f"  coll: start->buf_ready {d(2, 1):.0f}  buf_ready->polled {d(3, 2):.0f}  polled->posted {d(4, 3):.0f}"
          f"  posted->next start {np.median(x[sl, 1][1:] - x[sl, 4][:-1]):.0f}")
    print(f"  own pub(q)->coll_start(q) {d(1, 0):.0f}  pub(q)->posted(q) {d(4, 0):.0f}")
    print(f"  consumer wait for g(q): {d(6, 5):.0f}  pub(q+2)->cons_wait(q) {np.median(x[sl, 5][:-2] - x[sl, 0][2:]):.0f}")
    print(f"  re-poll rounds: mean {x[sl, 7].mean():.2f} max {x[sl, 7].max():.0f}")
