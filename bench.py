#!/usr/bin/env python
"""AM-QFT benchmark (BASELINE.json config 2 by default).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch: a batched complex fp32
forward DFT, N=4096, batch=65536 (2 GiB in + 2 GiB out, interleaved re/im,
iid N(0,1) from a seed), AM-QFT variant 4 (the improved QFT) by default.
Inputs are resident in HBM when the timed region starts and are 16x larger
than L2, so no flush is needed between steps.  Multi-GPU (torchrun): every
rank runs its own 65536-transform shard (weak scaling, no communication);
time = max over ranks of the CUDA-event time.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libamqft_ref.so: the unmodified reference library compiled from
its sources) on the host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AM-QFT transforms/s (CDFT N=4096 fp32, batch 65536)"
UNIT = "transforms/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--variant", type=int, default=4)
    p.add_argument("--n", type=int, default=4096)
    p.add_argument("--batch", type=int, default=65536)
    p.add_argument("--dtype", default="f32")
    p.add_argument("--order", choices=["fast", "exact"], default="fast")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--all-variants", action=argparse.BooleanOptionalAction, default=True,
                   help="after the timed region, also time variants 1..8 and report their fp32 error "
                        "(extra 'variants' and accuracy keys; --no-all-variants to skip)")
    p.add_argument("--strong", action="store_true",
                   help="config 2 strong scaling: the fixed batch is sharded by global row over the ranks "
                        "(default: weak scaling, every rank runs its own full batch)")
    p.add_argument("--config", type=int, choices=[2, 4, 5], default=2,
                   help="BASELINE config: 2 batched N=4096 (default), 4 single N=2^24 four-step, "
                        "5 single N=2^30 distributed four-step over the ranks")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [s.strip() for s in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(args, seconds_target=10.0):
    """Reference CPU path (oracle/_ref) on the host cores, bounded sample of the
    same workload (fp32 inputs widened to double: the reference is fp64-only)."""
    import numpy as np
    from oracle import oracle as O
    ref = O.reference()
    kind = "reference"
    if ref is None:  # reference never compiled: the C restatement stands in
        ref = O.restatement()
        kind = "port"
    threads = os.cpu_count() or 1
    n = args.n
    rng = np.random.default_rng(1234)

    def run(rows):
        x = rng.standard_normal((rows, 2 * n)).astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        if kind == "reference":
            ref.execute_rows(args.variant, O.CDFT, n, x, threads)
        else:
            for r in range(rows):
                ref.execute(args.variant, O.F_CDFT, n, x[r])
        return time.perf_counter() - t0

    probe = max(threads, 8)
    dt = run(probe)
    rate = probe / dt
    rows = int(min(max(probe, rate * seconds_target), 200000))
    dt = run(rows)
    value = rows / dt
    used = threads if kind == "reference" else 1
    return {"value": value, "unit": UNIT, "cores": used, "kind": kind,
            "sample": f"{rows} rows of CDFT N={n} (variant {args.variant}), fp32 data widened to fp64, "
                      f"{used} threads, {dt:.1f} s",
            "gbs_fp32_bytes": value * 16 * n / 1e9, "gbs_fp64_bytes": value * 32 * n / 1e9}


def bench_reference(args, rank):
    """--impl reference: the reference's own CPU implementation, rank 0 only.
    One step = the reference library (oracle/_ref) over a fixed sample of
    rows of the config-2 workload on every host thread; the sample is sized
    once in the warm-up (~2 s per step), then every timed step runs exactly
    that many rows and its wall time is measured."""
    if rank != 0:
        return None
    import numpy as np
    from oracle import oracle as O
    ref = O.reference()
    kind = "reference"
    if ref is None:  # reference never compiled: the C restatement stands in
        ref, kind = O.restatement(), "port"
    threads = os.cpu_count() or 1
    n = args.n
    x = np.random.default_rng(1234).standard_normal((max(threads, 8), 2 * n)).astype(np.float32).astype(np.float64)

    def step(rows):
        xs = np.resize(x, (rows, 2 * n))
        t0 = time.perf_counter()
        if kind == "reference":
            ref.execute_rows(args.variant, O.CDFT, n, xs, threads)
        else:
            for r in range(rows):
                ref.execute(args.variant, O.F_CDFT, n, xs[r])
        return time.perf_counter() - t0

    probe = max(threads, 8)
    rate = probe / step(probe)
    rows = int(min(max(probe, rate * 2.0), args.batch))
    for _ in range(max(0, args.warmup - 1)):
        step(rows)
    times = [step(rows) for _ in range(args.steps)]
    step_s = statistics.mean(times)
    value = rows / step_s
    used = threads if kind == "reference" else 1
    cb = {"value": value, "unit": UNIT, "cores": used, "kind": kind,
          "sample": f"{rows} rows of CDFT N={n} (variant {args.variant}) per step, fp32 data widened to fp64, "
                    f"{used} threads; {args.steps} steps, mean {step_s:.2f} s",
          "gbs_fp32_bytes": value * 16 * n / 1e9, "gbs_fp64_bytes": value * 32 * n / 1e9}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * step_s, "rows_per_step": rows, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) (seeded), fp32 values widened to fp64",
        "config": {"workload": f"config 2: batched CDFT N={args.n} x {args.batch}, variant {args.variant} "
                               f"(each step a {rows}-row sample)",
                   "n": args.n, "batch": args.batch, "variant": args.variant,
                   "parallelism": "host threads"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def ncu_traffic(args, n, path=2):
    """DRAM bytes per launch of the timed kernel from the committed ncu
    --set full capture (profiles/, made by tools/profile_round.sh), when it
    is a capture of this exact kernel (variant, N, fp32, fast order): k_tile
    (path 6, the in-shared-memory four-step) or k_fast (path 2)."""
    import glob
    logn = n.bit_length() - 1
    if args.dtype != "f32" or args.order != "fast":
        return None, None
    if path == 6:
        # k_tile<V, R, INV, TCfg<R, LG1, LG2, ...>>: N1 x N2 = 64 x 64 at N = 4096 (tile_kernel.cuh make_tile)
        lg1 = 6 if logn == 11 else logn // 2
        want = tuple(f"k_tile<{args.variant},float,{b},TCfg<float,{lg1},{logn - lg1}," for b in ("false", "0"))
        pattern = "r*_ncu_k_tile_*.json"
    else:
        # k_fast<V, R, LOGN, LOGLB, MODE[, IO, P]>: the one-CTA-per-row fp32 instance
        want = (f"k_fast<{args.variant},float,{logn},6,0>", f"k_fast<{args.variant},float,{logn},6,0,float,1>")
        pattern = "r*_ncu_k_fast_*.json"
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)), reverse=True):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        name = d.get("Kernel Name", "")
        for junk in (" ", "(bool)", "(int)", "amqft_b200::tilek::", "amqft_b200::fastk::"):
            name = name.replace(junk, "")
        if not any(w in name for w in want) or int(float(d.get("launch__grid_size", 0))) <= 0:
            continue
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1.0}
        rd = float(d["dram__bytes_read.sum"]) * scale.get(d.get("dram__bytes_read.sum [unit]", "Gbyte"), 1e9)
        wr = float(d["dram__bytes_write.sum"]) * scale.get(d.get("dram__bytes_write.sum [unit]", "Gbyte"), 1e9)
        return rd + wr, os.path.relpath(f, ROOT)
    return None, None


CHUNK = 512   # rows per generator chunk


def gen_rows(row0, rows, n, dtype, dev, seed=20260):
    """Rows [row0, row0 + rows) of the synthetic config-2 batch, iid N(0,1):
    counter-based by 512-row chunk (a Philox torch.Generator seeded with
    seed + chunk index), so a row's values depend only on its global index,
    never on how the batch is sharded over ranks."""
    import torch
    out = torch.empty(rows, 2 * n, dtype=dtype, device=dev)
    g = torch.Generator(device=dev)
    c0, c1 = row0 // CHUNK, (row0 + rows + CHUNK - 1) // CHUNK
    for c in range(c0, c1):
        g.manual_seed(seed + c)
        blk = torch.randn(CHUNK, 2 * n, generator=g, device=dev, dtype=dtype)
        lo, hi = max(row0, c * CHUNK), min(row0 + rows, (c + 1) * CHUNK)
        out[lo - row0:hi - row0] = blk[lo - c * CHUNK:hi - c * CHUNK]
    return out


def _timed(fn, steps, warmup, stream, world, dev):
    import torch
    import torch.distributed as dist
    for _ in range(max(warmup, 3)):
        fn()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms / steps


def cpu_baseline_large(variant, n_full, sample_n, seconds_cap=30.0):
    """Bounded CPU sample for the single-transform configs: one transform at
    a smaller N with the reference library, extrapolated by N log N."""
    import numpy as np
    from oracle import oracle as O
    ref = O.reference()
    kind = "reference"
    if ref is None:
        ref, kind = O.restatement(), "port"
    x = np.random.default_rng(7).standard_normal(2 * sample_n)
    t0 = time.perf_counter()
    if kind == "reference":
        ref.execute_rows(variant, O.CDFT, sample_n, x.reshape(1, -1), 1)
    else:
        ref.execute(variant, O.F_CDFT, sample_n, x)
    dt = time.perf_counter() - t0
    lg_s, lg_f = sample_n.bit_length() - 1, n_full.bit_length() - 1
    est = dt * (n_full * lg_f) / (sample_n * lg_s)
    return {"value": 1.0 / est, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"one CDFT N=2^{lg_s} (variant {variant}) in {dt:.1f} s on 1 thread (one transform does not "
                      f"parallelise in the reference), extrapolated to N=2^{lg_f} by N log N: {est:.0f} s"}


def oracle_checks(args, kept, amqft, kept_v=None):
    """Checker only (runs in the CPU-baseline leg)."""
    import numpy as np
    from oracle import oracle as O
    r = O.restatement()
    n = args.n
    parity = max(r.rel_l2(got, r.execute(args.variant, O.F_CDFT, n, xin)) for xin, got in kept)
    acc = {}
    n1 = 1024
    x1 = O.seeded_signal(1, O.CDFT, n1, 0, r)      # config 1: U[-1,1), mix_seed(1, kind, n, trial)
    naive = r.naive(O.CDFT, n1, x1)
    for v in range(1, 9):
        got = amqft.execute(v, amqft.FunctionId.Cdft, n1, x1)
        acc[str(v)] = {
            "bitwise_vs_cpu_same_variant": bool(got.tobytes() == r.execute(v, O.F_CDFT, n1, x1).tobytes()),
            "rel_l2_vs_naive_fp64": r.rel_l2(got, naive),
            "rel_l2_vs_extended": r.rel_error_extended(O.CDFT, n1, x1, got),
        }
    out = {"config1_fp64_n1024": acc}
    if kept_v:
        out["config2_fp32_row0_rel_l2_vs_cpu_same_variant"] = {
            str(v): r.rel_l2(got, r.execute(v, O.F_CDFT, n, xin)) for v, (xin, got) in sorted(kept_v.items())}
        xin0 = next(iter(kept_v.values()))[0]
        naive_n = r.naive(O.CDFT, n, xin0)      # O(N^2) fp64 DFT of the same row (BASELINE)
        out["config2_fp32_row0_rel_l2_vs_naive_fp64"] = {
            str(v): r.rel_l2(got, naive_n) for v, (xin, got) in sorted(kept_v.items()) if xin is xin0 or
            np.array_equal(xin, xin0)}
        out["config2_tolerance_fp32"] = 1e-5 * math.log2(n)
    return parity, out


def config4_accuracy(amqft, x, n, local, stream, args):
    """BASELINE config 4: every variant's fp32 result against an fp64 result
    of the same input, with the tabulated and the on-the-fly half-size
    twiddle sets.  The fp64 result is the GPU fp64 four-step of variant 4
    (sub-transforms bitwise the reference recursion), itself checked
    against numpy's fp64 FFT (C4 is beyond a timely CPU
    oracle)."""
    import numpy as np
    import torch
    ref = amqft.Plan(4, amqft.FunctionId.Cdft, n, 1, dtype="f64", order=amqft.Order.Fast, device=local)
    xd = x.double()
    y64 = torch.empty_like(xd)
    ref.forward(xd, y64, stream=stream)
    torch.cuda.synchronize()
    xh = xd[0].cpu().numpy()
    f = np.fft.fft(xh[0::2] + 1j * xh[1::2])
    fh = np.empty(2 * n)
    fh[0::2], fh[1::2] = f.real, f.imag
    yh = y64[0].cpu().numpy()
    out = {"reference": "GPU fp64 four-step, variant 4",
           "reference_vs_numpy_fft_rel_l2": float(np.linalg.norm(yh - fh) / np.linalg.norm(fh))}
    del ref
    y = torch.empty_like(x)
    for trig, key in ((amqft.TrigMode.Precomputed, "table"), (amqft.TrigMode.OnTheFly, "onthefly")):
        errs = {}
        for v in range(1, 9):
            p = amqft.Plan(v, amqft.FunctionId.Cdft, n, 1, dtype="f32", order=amqft.Order.Fast, trig_mode=trig,
                           device=local)
            p.forward(x, y, stream=stream)
            torch.cuda.synchronize()
            e = float((y.double() - y64).norm() / y64.norm())
            errs[str(v)] = e if math.isfinite(e) else str(e)
            if v == args.variant:
                out[f"ms_{key}"] = _timed(lambda: p.forward(x, y, stream=stream), 5, 2, stream, 1, torch.device(f"cuda:{local}"))
            del p
        out[f"rel_l2_fp32_vs_fp64_{key}"] = errs
    # direct spot checks (csrc/verify.cu): 64 bins of the fp64 reference and
    # of the timed variant's fp32 result against their O(N) fp64 sums
    bins = spot_bins(n, seed=24)
    want = amqft.direct_bins(x, n, bins, stream=stream)
    idx = torch.as_tensor(bins.astype(np.int64), device=x.device)

    def pick(t):
        c = t.view(-1, 2)[idx].double().cpu().numpy()
        return c[:, 0] + 1j * c[:, 1]
    p = amqft.Plan(args.variant, amqft.FunctionId.Cdft, n, 1, dtype="f32", order=amqft.Order.Fast, device=local)
    p.forward(x, y, stream=stream)
    torch.cuda.synchronize()
    out["spot_bins"] = {"bins": int(len(bins)),
                        "fp64_reference_rel_l2": float(np.linalg.norm(pick(y64) - want) / np.linalg.norm(want)),
                        f"fp32_v{args.variant}_rel_l2": float(np.linalg.norm(pick(y) - want) / np.linalg.norm(want))}
    out["tolerance_fp32"] = 1e-5 * 24
    return out


def spot_bins(n, count=64, seed=1):
    """Bins for the direct spot checks: the edges plus seeded random bins."""
    import numpy as np
    rng = np.random.default_rng(seed)
    edge = [0, 1, 2, n // 4, n // 2 - 1, n // 2, n // 2 + 1, n - 1]
    return np.unique(np.concatenate([edge, rng.integers(0, n, count - len(edge))])).astype(np.uint64)


def config5_spot_check(amqft, d, a0, bufs, stream, world, rank, dev):
    """Config 5 accuracy: 64 output bins of one more forward
    against their direct O(N) sums over the 2^30 input samples on the device
    (amqft_direct_bins: fp64, exact integer phase reduction), after the timed
    region.  Multi-rank: each rank sums its input slab, the partial bins are
    all-reduced, and the rank holding a bin's k1-slab reports it."""
    import numpy as np
    import torch
    import torch.distributed as dist
    n = d.n
    bins = spot_bins(n, seed=30)
    a = a0.clone()
    z = d.forward(a, bufs=bufs, stream=stream)
    torch.cuda.synchronize(dev)
    part = amqft.direct_bins(a0, n, bins, rows=d.rows1, row_len=d.n1, row0=rank * d.rows1, stride=d.n2,
                             stream=stream)
    want = torch.tensor(np.stack([part.real, part.imag], 1), dtype=torch.float64, device=dev)
    k1 = (bins % d.n1).astype(np.int64)
    k2 = (bins // d.n1).astype(np.int64)
    mine = (k1 // d.w) == rank
    got = torch.zeros(len(bins), 2, dtype=torch.float64, device=dev)
    if mine.any():
        zz = z.view(d.w, d.n2, 2)
        idx = np.nonzero(mine)[0]
        got[torch.as_tensor(idx, device=dev)] = zz[torch.as_tensor(k1[idx] - rank * d.w, device=dev),
                                                   torch.as_tensor(k2[idx], device=dev)].double()
    if world > 1:
        dist.all_reduce(want)
        dist.all_reduce(got)
    w = want.cpu().numpy()
    g = got.cpu().numpy()
    wc, gc = w[:, 0] + 1j * w[:, 1], g[:, 0] + 1j * g[:, 1]
    return {"spot_bins": int(len(bins)),
            "rel_l2_vs_direct_fp64_sums": float(np.linalg.norm(gc - wc) / np.linalg.norm(wc)),
            "max_abs_err_over_rms_bin": float(np.max(np.abs(gc - wc)) / np.sqrt(np.mean(np.abs(wc) ** 2))),
            "tolerance_1e-5_log2N": 3e-4,
            "method": "direct fp64 sums over all 2^30 samples per bin, phase (n k) mod N in 64-bit integers "
                      "(csrc/verify.cu), 64 bins incl. 0, 1, N/4, N/2, N-1"}


def bench_single(args, world, rank, local):
    """Configs 4 (N=2^24, one GPU, four-step) and 5 (N=2^30, distributed
    four-step over the ranks, one all-to-all)."""
    import torch
    import torch.distributed as dist
    import paper_1404_1810_b200 as amqft
    from paper_1404_1810_b200.dist import DistFourStep
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    hbm, hbm_src = peaks()
    g = torch.Generator(device=dev)
    g.manual_seed(4242 + rank)
    extra = {}
    if args.config == 4:
        n = 1 << 24
        # tabulated half-size twiddle set (two fp64 tables seed each thread's recurrence): as accurate as
        # the on-the-fly set and, on the column-slab passes, 2 % faster (both timed and reported in "accuracy")
        plan = amqft.Plan(args.variant, amqft.FunctionId.Cdft, n, 1, dtype="f32", order=amqft.Order.Fast,
                          trig_mode=amqft.TrigMode.Precomputed, device=local)
        x = torch.randn(1, 2 * n, generator=g, device=dev)
        y = torch.empty_like(x)
        ms = _timed(lambda: plan.forward(x, y, stream=stream), args.steps, args.warmup, stream, world, dev)
        path, launches = plan.path()
        fa, fb, fc = plan.fourstep_factors()
        shape = f"three-factor {fa} x {fb} x {fc}" if fb > 1 else f"two-factor {fa} x {fc}"
        # one launch per factor: the column-slab plan (no transposes); else column passes + rows + transpose
        slab = launches == (3 if fb > 1 else 2)
        kind = ("column-slab passes, natural order in and out, no transpose" if slab
                else "column passes + tile-kernel rows + one transpose")
        workload = (f"config 4: one complex forward DFT N=2^24 fp32, four-step {shape} ({kind}), "
                    f"tabulated twiddles, variant {args.variant}")
        per_gpu_bytes = 16 * n
        value = world / (ms / 1000.0)
        hx = torch.empty(1, 2 * n, pin_memory=True)
        hx.copy_(x)
        hy = torch.empty_like(hx, pin_memory=True)
        plan.forward_host(hx, hy, stream=stream)
        e2e_ms = _timed(lambda: plan.forward_host(hx, hy, stream=stream), 3, 1, stream, world, dev)
        e2e = {"value": world / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n}
        # every launch reads and writes the whole signal once
        extra = {"hbm_passes": launches, "traffic_model_bytes": launches * 16 * n,
                 "factors": [fa, fb, fc]}
        try:   # measured DRAM bytes per step (ncu, profiles/r02_ncu_c4_passes.json)
            prof = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_c4_passes.json")))
            if args.variant == 4 and len(prof["launches"]) == launches:
                extra["traffic_step_bytes"] = prof["step_dram_bytes"]
                extra["traffic_source"] = "profiles/r02_ncu_c4_passes.json"
        except (OSError, ValueError, KeyError):
            pass
        if rank == 0:
            extra["accuracy"] = config4_accuracy(amqft, x, n, local, stream, args)
        cpu = cpu_baseline_large(args.variant, n, 1 << 20) if (rank == 0 and not args.no_cpu_baseline) else None
    else:
        n = 1 << 30
        d = DistFourStep(args.variant, n, device=local, trig_mode=amqft.TrigMode.OnTheFly)
        # each rank generates its own column slab on the device (config 5)
        a0 = torch.randn(d.rows1, 2 * d.n1, generator=g, device=dev)
        a = torch.empty_like(a0)
        bufs = d.buffers(a0)

        def step():
            a.copy_(a0)
            d.forward(a, bufs=bufs, stream=stream)
        ms = _timed(step, args.steps, args.warmup, stream, world, dev)
        copy_ms = _timed(lambda: a.copy_(a0), args.steps, 1, stream, world, dev)
        a2a_ms = None
        if world > 1:
            a2a_ms = _timed(lambda: dist.all_to_all_single(bufs[1], bufs[0]), args.steps, 1, stream, world, dev)
        sent = (world - 1) * d.rows1 * d.w * 8
        ms = ms - copy_ms        # the slab refresh is not part of the transform
        # our kernels per step: the local length-n1 plan (its final transpose
        # folded into the scatter when it runs transposed), the twiddle-scatter,
        # the transpose, the length-n2 plan
        l1 = d.ops.p1.path()[1] - (1 if d.ops.a_t else 0)
        # one GPU: no exchange to make, the scatter writes each value to its final place (scatter +
        # transpose in one kernel: DistFourStep.forward's direct mode); several: scatter, all-to-all, transpose
        direct = world == 1 and d.ops.direct_ok(d.rows1)
        path, launches = 3, l1 + (1 if direct else 2) + d.ops.p2.path()[1]
        exch = "direct twiddle-scatter into the row buffer (no exchange on one GPU)" if direct else "one all-to-all"
        workload = (f"config 5: one complex forward DFT N=2^30 fp32 over {world} GPU(s), distributed four-step "
                    f"n1=2^{d.n1.bit_length() - 1} x n2=2^{d.n2.bit_length() - 1}, {exch}, on-the-fly twiddles, "
                    f"variant {args.variant}")
        per_gpu_bytes = 16 * n // world
        value = 1.0 / (ms / 1000.0)
        e2e = None
        extra = {"a2a_ms": a2a_ms, "a2a_bytes_sent_per_gpu": sent,
                 "nvlink_frac": (sent / (a2a_ms / 1000.0) / 900e9) if a2a_ms else None,
                 "output_layout": "k1-slabs (rows k1 of length n2 per rank); no second all-to-all",
                 "accuracy": config5_spot_check(amqft, d, a0, bufs, stream, world, rank, dev)}
        cpu = None
    achieved = per_gpu_bytes / (ms / 1000.0) / 1e9
    if rank == 0:
        line = {
            "metric": f"AM-QFT transforms/s ({'N=2^24' if args.config == 4 else 'N=2^30'} fp32 single transform)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic: iid N(0,1) from a seed, generated on the device",
            "config": {"workload": workload, "n": n, "variant": args.variant, "path": path,
                       "l2": "inputs >= 128 MiB > 126 MB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": extra.get("traffic_step_bytes"), "peak_source": hbm_src,
                         "algorithmic_bytes_per_gpu": per_gpu_bytes},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches * args.steps if launches is not None else None,   # inside the timed region
            "launches_per_step": launches, **extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config in (4, 5) and args.impl == "ours":
        bench_single(args, world, rank, local)
        return

    if args.impl == "reference":
        line = bench_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_1404_1810_b200 as amqft

    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n = args.n
    # weak (default): every rank runs a full batch of its own rows; strong
    # (--strong): the fixed batch sharded by global row
    if args.strong:
        if args.batch % world:
            raise SystemExit("--strong: the batch must divide over the ranks")
        batch = args.batch // world
        row0 = rank * batch
    else:
        batch = args.batch
        row0 = rank * batch
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    esize = 4 if args.dtype == "f32" else 8
    order = amqft.Order.Fast if args.order == "fast" else amqft.Order.Exact
    plan = amqft.Plan(args.variant, amqft.FunctionId.Cdft, n, batch, dtype=args.dtype,
                      order=order, device=local)
    path, launches = plan.path()
    x = gen_rows(row0, batch, n, dtype, dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 3)):
        plan.forward(x, y, stream=stream)
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.forward(x, y, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * batch * args.steps / (ms / 1000.0)

    # Dominant-kernel roofline: the exec call is one kernel on paths 0/2/6;
    # per-launch duration from CUDA events on the launching stream.
    hbm, hbm_src = peaks()
    alg_bytes = 2 * (2 * n * esize) * batch  # one read + one write per transform
    kernel_ms = ms_per_step / max(1, launches) if path != 1 else ms_per_step
    achieved = alg_bytes / (kernel_ms / 1000.0) / 1e9
    traffic, traffic_src = ncu_traffic(args, n, path)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read + write)",
            "traffic_source": traffic_src,
            "peak_source": hbm_src, "algorithmic_bytes_per_launch": alg_bytes,
            "kernel_ms": kernel_ms}

    # Parity of what was timed (checked in the CPU-baseline leg below, the
    # one place the oracle runs): keep a few output rows on the host.
    check_rows = (0, batch // 2, batch - 1)
    kept = [(x[row].double().cpu().numpy(), y[row].double().cpu().numpy()) for row in check_rows]
    parity = None

    # End to end through the public API with HOST buffers (pinned): H2D of the
    # step's input, the transform, D2H of the result, every step.
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.empty(batch, 2 * n, dtype=dtype, pin_memory=True)
        hx.copy_(x)
        hy = torch.empty_like(hx, pin_memory=True)
        plan.forward(x, y, stream=stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        plan.forward_host(hx, hy, stream=stream)   # creates the pipeline slots (untimed)
        torch.cuda.synchronize(dev)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.e2e_steps):
            # public host-buffer entry point: H2D | transform | D2H pipelined
            plan.forward_host(hx, hy, stream=stream)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        ems = torch.tensor([s0.elapsed_time(s1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": world * batch * args.e2e_steps / (float(ems.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": batch * 2 * n * esize, "d2h_bytes_per_step": batch * 2 * n * esize,
               "steps": args.e2e_steps}

    variants = None
    kept_v = {}
    if args.all_variants:
        variants = {}
        for v in range(1, 9):
            pv = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype=args.dtype, order=order,
                            device=local)
            for _ in range(3):
                pv.forward(x, y, stream=stream)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                pv.forward(x, y, stream=stream)
            b.record(stream)
            torch.cuda.synchronize(dev)
            vms = a.elapsed_time(b) / args.steps
            variants[str(v)] = {"transforms_per_s": batch / (vms / 1000.0), "ms": vms,
                                "gbs": alg_bytes / (vms / 1000.0) / 1e9}
            kept_v[v] = (x[0].double().cpu().numpy(), y[0].double().cpu().numpy())
            pv.close()

    cpu = None
    accuracy = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"failed: {e}"}
        # CPU leg, checker use of the oracle: parity of the timed rows, and
        # every variant's config-1 accuracy (N = 1024 fp64 exact path on the
        # device) against the reference CPU result, the naive O(N^2) fp64
        # DFT and the extended-precision spectrum (north_star reporting)
        try:
            parity, accuracy = oracle_checks(args, kept, amqft, kept_v)
        except Exception as e:  # noqa: BLE001
            parity = f"unavailable: {e}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": args.dtype,
            "data": "synthetic: iid N(0,1), counter-based per 512-row chunk of the global batch (Philox)",
            "config": {"workload": f"config 2: batched complex forward DFT N={n}, "
                                   + (f"batch {args.batch} sharded over {world} GPU(s) by global row"
                                      if args.strong else f"batch {batch} per GPU")
                                   + f", interleaved re/im, AM-QFT variant {args.variant}",
                       "n": n, "batch_per_gpu": batch, "global_batch": batch * world, "variant": args.variant,
                       "order": args.order, "path": path, "launches_per_step": launches,
                       "l2": f"inputs {batch * 2 * n * esize / 2**30:.2f} GiB per GPU > 126 MB L2; no flush",
                       "parallelism": f"batch-sharded x{world}, no communication"},
            "gbs": alg_bytes * world / (ms_per_step / 1000.0) / 1e9,
            "per_gpu": {"transforms_per_s": value / world, "gbs": alg_bytes / (ms_per_step / 1000.0) / 1e9,
                        "frac_of_n_x_hbm": (alg_bytes * world / (ms_per_step / 1000.0) / 1e9) / (world * hbm)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
            "parity_rel_l2_vs_cpu_same_variant": parity,
            "accuracy": accuracy,
        }
        if variants:
            line["variants"] = variants
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
