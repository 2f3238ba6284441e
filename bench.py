#!/usr/bin/env python
"""DXG benchmark: iterations/s at n=1e5 with the FP64 cost matrix stored in HBM.

Workload (BASELINE.json configs[2], the configuration the metric is quoted on):
n = 100,000, C_ij = splitmix64(seed, i, j) -> U[0,1) generated in HBM (80 GB),
random r, c (seeded), params_tuned(0) with tau_mu = 0.05.  One
step = one DXG iteration (dxg_step): both column marginals (pass A + pass B over
C) + the fused O(n) updates.  C (80 GB) is far larger than L2 (126 MB), so every
iteration streams it from HBM; no L2 flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 is launched by torchrun (one rank per GPU, NCCL): rows are sharded, the
2n column partials are all-gathered every iteration (strong scaling: total work
fixed).  `--impl reference` times the reference algorithm on the host cores
(oracle/ port of leanot; bounded sample of rows, extrapolated per iteration).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DXG iters/s and time-to-ε at n=1e5 FP64 (% roofline), 1/2/4/8 B200 vs CPU"
UNIT = "iters/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FP64_PEAK_DFMA = 17.07e12       # measured DFMA/s on this pool's B200 (profiles/r01_microbench.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the config-4 shard (FP64-bound path) timing")
    ap.add_argument("--no-tte", action="store_true", help="skip the config-1 time-to-eps run")
    return ap.parse_args()


def marginals(n, seed):
    rng = np.random.default_rng(seed + 1)
    r = rng.random(n)
    c = rng.random(n)
    return r / r.sum(), c / c.sum()


def hbm_peak():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap,enforced.power.limit", "--format=csv,noheader,nounits",
                 "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons, pw, lim = [], 0.0, set(), [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
                lim = float(parts[7])
            except (ValueError, IndexError):
                pass
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            out["power_w"] = statistics.median(pw)     # board power during the timed region
            out["power_limit_w"] = lim
        return out


# ---------------------------------------------------------------------------
# CPU reference (oracle port of leanot) -- bounded sample, extrapolated
# ---------------------------------------------------------------------------


def cpu_reference(n, seed, steps, warmup):
    """Times the reference's per-iteration work (both column_marginal sweeps of
    dxg_step, dxg.py:193-208, 272-276) on a sample of rows with all host threads."""
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import leanot_oracle as O
    cores = O.default_workers()
    rows = O.BLOCK_ROWS * cores          # one 128-row block per thread
    rows = min(rows, n)
    cost = O.HashCost(n, seed)
    blocks = [cost.block(i0, min(i0 + O.BLOCK_ROWS, rows)) for i0 in range(0, rows, O.BLOCK_ROWS)]
    r, c = marginals(n, seed)
    prm = O.params_tuned(0.0, tau_mu=0.05)
    rng = np.random.default_rng(seed + 7)
    it = O.Iterate(rng.uniform(-1, 1, n), 40.0, -np.abs(rng.normal(0, 20, n)), 0.0, 40)
    a_bar, b_bar, _, _ = O._advance(it.a, it.b, it.s, it.t, np.tanh(0.5 * it.delta), prm, 1.0)
    wsets = [(it.a, it.b), (a_bar, b_bar)]

    class Sample:
        def __init__(self):
            self.n = n

        def block(self, i0, i1):
            return blocks[i0 // O.BLOCK_ROWS]

    sample = Sample()

    def one():
        # dxg_step runs column_marginal twice, each a full pass over the blocks
        # (dxg.py:272, :276; column_marginal dxg.py:193-208), so the two weight sets are two
        # separate passes here too (no shared block read)
        t0 = time.perf_counter()
        for a, b in wsets:
            def work(i0, i1, a=a, b=b):
                return r[i0:i1] @ O._softmax_block(a, b, sample.block(i0, i1))
            O.run_blocks(work, rows, workers=cores)
        return time.perf_counter() - t0

    for _ in range(warmup):
        one()
    times = [one() for _ in range(steps)]
    per_iter = statistics.median(times) * (n / rows)
    return {"value": 1.0 / per_iter, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{rows} of {n} rows of C (both column_marginal passes of one dxg_step, one 128-row "
                      f"block per thread, {cores} threads, numpy {np.__version__}), median of {steps} steps, "
                      f"scaled x{n / rows:.1f} to one iteration (the full iteration is ~{n / rows:.0f}x the sample)",
            "seconds_per_iter": per_iter}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def init_dist(args):
    """One process per GPU (torchrun env).  LEANOT_BENCH_BACKEND=gloo (tests only) runs the ranks
    on whatever GPUs exist, possibly all on one, with host-staged collectives."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("LEANOT_BENCH_BACKEND", "nccl")
    dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    return world, rank, dev, group


def barrier(group):
    if group is not None:
        import torch.distributed as dist
        dist.barrier(group=group)


def max_over_ranks(x, group):
    if group is None:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def time_to_eps_config1():
    """BASELINE config 1 end to end on the GPU (reference: 8,225 iterations)."""
    import torch
    from paper_2511_11359_b200 import core, dxg
    n = 1000
    rng = np.random.default_rng(0)
    r = core.Histogram.normalized(rng.random(n))
    c = core.Histogram.normalized(rng.random(n))
    k = core.ExplicitKernel(rng.random((n, n)))
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4, max_iter=50), dense_cap=0)  # warm (graphs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = dxg.solve(k, r, c, prm, dxg.Termination(eps=1e-4), log_stride=25, dense_cap=0)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    return {"config": "n=1000 random C, tuned+tau_mu=0.05, eps=1e-4 (BASELINE config 1)",
            "seconds": secs, "iterations": sol.iterations, "converged": sol.converged,
            "reference_iterations": 8225, "reference_seconds_published": None,
            "reference_seconds_survey_4workers": 93.0}


def fp64_path_config4(iters=2):
    """BASELINE config 4's per-GPU work (one 1/8 row shard of n=1e6 3-D points, cost on the fly)
    timed in this run: the FP64-bound path's roofline (north_star: >= 70 % of the FP64 roofline
    for on-the-fly C).  Same engine calls as tools/bench_configs.py config4."""
    import torch
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import DxgEngine, shard_rows
    n, shards = 1_000_000, 8
    rng = np.random.default_rng(4)
    f = rng.random((n, 3))
    f[0], f[1] = 0.0, 1.0            # cube corners: raw sup = 3 by construction
    k = core.ColorKernel(f, 2, scale=3.0)
    r0, r1 = shard_rows(n, shards, 0)
    k.row0, k.row1 = r0, r1
    w1, w2 = rng.random(n), rng.random(n)
    eng = DxgEngine(k, w1 / w1.sum(), w2 / w2.sum(), dxg.params_tuned(1e-7).with_overrides(tau_mu=0.05))
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    eng.sweep()
    eng.update()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(iters):
        eng.sweep()
        eng.update()
    e1.record(st)
    torch.cuda.synchronize()
    per_iter = e0.elapsed_time(e1) / 1e3 / iters
    elems = n * (r1 - r0)
    executed = 2 * (3 + 2 * 8)   # per element and iteration: 2 passes x (3-term dot + 2 sets x (x' + 7 exp))
    peak = 17.07e12              # builder DFMA microbenchmark at 1965 MHz (profiles/r01_microbench.md)
    return {"what": "BASELINE config 4 per-GPU work: one 1/8 row shard of n=1e6 3-D points (cost on the fly, "
                    "expanded form), DXG iteration, measured in this run (CUDA events)",
            "rows": r1 - r0, "n": n, "iters": iters, "seconds_per_iteration": per_iter,
            "fp64_instr_per_s_executed": executed * elems / per_iter,
            "frac_executed": executed * elems / per_iter / peak,
            "frac_survey_count": 47 * elems / per_iter / peak,
            "peak_fp64_instr_per_s": peak,
            "peak_source": "builder DFMA microbenchmark (tools/microbench/fp64_bench.cu, 17.07e12/s at 1965 MHz); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "definitions": "executed: 38 FP64 instructions per element and iteration the two-pass expanded-form "
                           "kernels issue; survey: SURVEY.md 8(d)'s 47 per element (libdevice exp count)"}


def run_b200(args):
    import torch
    world, rank, local, group = init_dist(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}, or plain `bench.py --gpus N`)")
    from paper_2511_11359_b200 import core, dxg
    from paper_2511_11359_b200.engine import DxgEngine, shard_rows

    n = args.n
    r0, r1 = shard_rows(n, world, rank)
    kern = core.HashKernel(n, seed=args.seed, rows=(r0, r1))
    r, c = marginals(n, args.seed)
    prm = dxg.params_tuned(0.0).with_overrides(tau_mu=0.05)
    eng = DxgEngine(kern, r, c, prm, group=group)
    eng.load_state(np.zeros(n), np.zeros(n), 0.0, 0.0, 0, fresh=True)
    nr = r1 - r0
    stream = torch.cuda.current_stream()
    for _ in range(max(3, args.warmup)):
        eng.sweep()
        eng.update()
    torch.cuda.synchronize()
    barrier(group)

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(group)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(K):
            e = evs[k]
            e[0].record(stream)
            eng.sweep_phase("rows")
            e[1].record(stream)
            eng.sweep_phase("cols")
            e[2].record(stream)
            eng.update()
            e[3].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier(group)
    elapsed = t_start.elapsed_time(t_end) / 1e3
    elapsed_max = max_over_ranks(elapsed, group)
    t_rows = [e[0].elapsed_time(e[1]) / 1e3 for e in evs]
    t_cols = [e[1].elapsed_time(e[2]) / 1e3 for e in evs]
    t_upd = [e[2].elapsed_time(e[3]) / 1e3 for e in evs]
    value = K / elapsed_max
    ms_per_step = 1e3 * elapsed_max / K

    peak, peak_kind = hbm_peak()
    bytes_alg = 8.0 * n * nr                       # one read of this rank's rows of C per iteration (per-GPU roofline)
    t_sweep = statistics.mean(t_rows) + statistics.mean(t_cols)
    # dominant kernel = pass B (column sums); report it and the whole sweep
    t_colk = statistics.mean(t_cols)
    fp64_per_elem = 2 * 8 + 2 * 8                  # 8 FP64 instr per element and weight set in each pass
    it_bytes_per_s = bytes_alg / (ms_per_step / 1e3)   # one read of C per iteration
    roofline = {
        "bound": "hbm", "what": "one DXG iteration: 8 n^2 algorithmic bytes (one read of C, SURVEY.md §8d) "
                                "/ ms_per_step",
        "achieved": it_bytes_per_s / 1e9, "peak": peak, "unit": "GB/s", "frac": it_bytes_per_s / 1e9 / peak,
        "peak_kind": peak_kind, "bytes_alg_per_iteration": bytes_alg,
        "traffic": None, "traffic_source": None,
        "dominant_kernel": {
            "kernel": "colpass_kernel<CostStored,2> (pass B, column sums of both weight sets)",
            "seconds_per_launch": t_colk, "bytes_alg_per_launch": bytes_alg,
            "achieved_gbs": bytes_alg / t_colk / 1e9, "frac": bytes_alg / t_colk / 1e9 / peak,
            "note": "per launch: each of the two passes reads C once, so the per-launch fraction "
                    "counts the second read as work; the iteration fraction above does not"},
        "limiter": "the two-pass sweep reads C twice and evaluates 4 exps per element; the board "
                   "sits at its 1 kW cap (sw_power_cap) running ~8 FP64 + 5 other instructions per exp "
                   "(profiles/r01_power.md); the single-read kernel (csrc/leanot_sr.cu, opt-in, 2 exps per "
                   "element) is bound by its consumer instruction stream (32 ms with the exchange and the "
                   "C copies disabled; profiles/r02/sr_instr_mix.md)",
        "sweep": {"what": "pass A + pass B (one DXG iteration's n^2 work)", "seconds": t_sweep,
                  "hbm_frac_vs_one_read": bytes_alg / t_sweep / 1e9 / peak,
                  "fp64_instr_per_s": fp64_per_elem * n * nr / t_sweep,
                  "fp64_frac_of_measured_dfma_peak": fp64_per_elem * n * nr / t_sweep / FP64_PEAK_DFMA,
                  "fp64_peak_source": "builder microbenchmark at 1965 MHz (profiles/r01_microbench.md), "
                                      "not MEASURED_PEAKS.json"},
        "phase_ms": {"rowpass": 1e3 * statistics.mean(t_rows), "colpass": 1e3 * t_colk,
                     "update": 1e3 * statistics.mean(t_upd)},
    }
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists() and world == 1:      # the capture is of the single-GPU (all rows) launch
        try:
            tj = json.loads(prof.read_text())
            roofline["traffic"] = tj.get("colpass_dram_bytes_per_launch")
            roofline["traffic_source"] = ("ncu --set full capture of the same kernel (profiles/traffic.json, "
                                          "separate run, not measured in this run): dram bytes read+write per "
                                          "pass-B launch")
        except Exception:
            pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": max(3, args.warmup),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (counter-based hash C in HBM, seeded random marginals)",
        "config": {"workload": "BASELINE config 3: n=1e5 stored FP64 cost (80 GB in HBM), DXG iteration",
                   "n": n, "rows_per_rank": nr, "params": "params_tuned(0) + tau_mu=0.05",
                   "l2": "inputs (80 GB) >> L2 (126 MB); no flush needed", "parallelism": f"row-shard x{world}"},
        "roofline": roofline,
        "gpu_launches": 7 * K,     # per iteration: rowpass, fixup, colpass, slab_reduce, 3 update kernels
    }
    clocks = clk.summary()
    if clocks:
        line["clocks"] = clocks

    # end to end through the public step API with host state (dxg.dxg_step)
    if not args.no_e2e:
        # the public step API with host state; under torchrun it sees the process group
        # (engine.default_group) and this rank's row shard of the cost
        kc = kern
        st = dxg.DxgState(dxg.LogOddsField(np.zeros(n)), dxg.TransportLogWeights(0.0, np.zeros(n), 0.0, 0))
        rh, ch = core.Histogram(r), core.Histogram(c)
        for _ in range(2):
            st = dxg.dxg_step(st, kc, rh, ch, prm)
        torch.cuda.synchronize()
        barrier(group)
        t0 = time.perf_counter()
        for _ in range(K):
            st = dxg.dxg_step(st, kc, rh, ch, prm)
        torch.cuda.synchronize()
        el = max_over_ranks(time.perf_counter() - t0, group)
        e2e = K / el
        line["e2e"] = {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                       "api": "paper_2511_11359_b200.dxg.dxg_step(state numpy in/out)"}
    if rank == 0 and world == 1 and not args.no_tte:
        try:
            line["time_to_eps"] = time_to_eps_config1()
        except Exception as e:  # report, do not hide
            line["time_to_eps"] = {"error": repr(e)}
        # the headline instance's time-to-eps takes 4.5-15 min (too long for this run): the
        # committed record of the same solver on the same instance, labelled as such
        rec = ROOT / "profiles" / "r02_tte_config3_eps1e-5.json"
        if not rec.exists():
            rec = ROOT / "profiles" / "r02_tte_config3_eps1e-4.json"
        if rec.exists():
            try:
                d = json.loads(rec.read_text())
                tr = d["trajectory_every_25"]
                hits = {}
                for eps in (1e-3, 1e-4, 1e-5):
                    h = [p for p in tr if abs(p[4]) <= eps / 6 and p[5] <= eps / 6]
                    if h:
                        hits[str(eps)] = {"iterations": h[0][0], "seconds": h[0][1]}
                line["time_to_eps_n1e5_recorded"] = {
                    "measured_in_this_run": False,
                    "source": f"profiles/{rec.name} (tools/tte_config3.py / tools/tte_resume.py, separate GPU "
                              "runs of the same solver; NOT measured in this run)",
                    "eps_1e-6": "not measured: ~7.8e5 iterations (~8 h) extrapolated from the 1e-4 -> 1e-5 "
                                "iteration ratio (4.38x)",
                    "instance": "BASELINE config 3 (n=1e5 stored C, tuned + tau_mu=0.05)", "eps": hits}
            except Exception as e:  # report, do not hide
                line["time_to_eps_n1e5_recorded"] = {"error": repr(e)}
    if world == 1 and not args.no_fp64:
        # the opt-in single-read sweep (one read of C, 2 exps per element) on the same engine,
        # timed after the headline region: what the north-star single-read design measures here
        try:
            for _ in range(2):
                eng.sweep(single_read=True)
                eng.update()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(5):
                eng.sweep(single_read=True)
                eng.update()
            ev1.record(stream)
            torch.cuda.synchronize()
            t_sr = ev0.elapsed_time(ev1) / 1e3 / 5
            line["single_read"] = {
                "what": "opt-in single-read sweep (csrc/leanot_sr.cu, default variant g) + update, 5 iterations "
                        "after the headline region, CUDA events",
                "ms_per_iteration": 1e3 * t_sr, "iters_per_s": 1.0 / t_sr,
                "hbm_frac_one_read": bytes_alg / t_sr / 1e9 / peak,
                "limiter": "consumer instruction stream (profiles/r02/sr_instr_mix.md); not the default path"}
        except Exception as e:  # report, do not hide
            line["single_read"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_fp64:
        try:
            line["fp64_path"] = fp64_path_config4()
        except Exception as e:  # report, do not hide
            line["fp64_path"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_reference(n, args.seed, steps=2, warmup=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if group is not None:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_reference(args.n, args.seed, steps=args.steps, warmup=max(1, min(args.warmup, 3)))
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * cb["seconds_per_iter"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based hash C regenerated on the host, seeded marginals)",
            "config": {"workload": "BASELINE config 3: n=1e5 stored FP64 cost, DXG iteration", "n": args.n},
            "impl": "reference", "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks (one process per
    GPU, NCCL) with torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    else:
        run_b200(a)
