"""GPU counterpart of the reference's `pafft bench` (tools/pafft_cli.cpp:35-62,
src/bench.cpp:128-311): times one operation on device-resident data and emits
the reference's table (same 10 columns, same FLOP/byte models) plus GPU
columns (batch, items/s, model GB/s, % of the measured HBM peak).

    python -m paper_2506_12718_b200.bench_ops --op conv-pa --radix 3 --dims 1594323 --batch 64
    python -m paper_2506_12718_b200.bench_ops --op all --radix 2 --dims 1048576

This reproduces the paper's per-operation split (permutation cost vs ladder
cost) on B200 and the permutation-avoiding vs standard-order
convolution comparison.  Inputs: SplitMix64 U(-1,1)
re/im from `--seed` (signal) and seed+1 (filter spectrum), as bench.cpp:135-147.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

OPS = ["permute", "fft", "fft-unordered", "ifft", "ifft-unordered", "conv-std", "conv-pa", "prepare-filter"]
HEADER = ["op", "radix", "dims", "total_n", "reps", "median_s", "min_s", "flop_est", "bytes_est", "ai_est"]
GPU_COLS = ["batch", "items_per_s", "model_gbs", "pct_hbm_peak", "precision"]


def parse_dims(text):
    """tools/pafft_cli.cpp:20-33: "64x64" -> [64, 64]."""
    dims = []
    for part in text.split("x"):
        if not part:
            raise ValueError(f"bad --dims value '{text}'")
        dims.append(int(part))
    return dims


def flop_bytes(op, n, radix, batch, esize):
    """bench.cpp:329-363 (per signal; x batch).  Radix 3/5 use the generic model."""
    from . import estimate_flop
    nd = float(n)
    fft_flop = estimate_flop(n, radix)
    logr = 0.0 if n < 2 else math.log2(nd) / math.log2(radix)
    full = 2.0 * nd * (1.0 + logr)
    bare = 2.0 * nd * logr
    if op in ("permute", "prepare-filter"):
        flop, elems = 0.0, 2.0 * nd
    elif op in ("fft", "ifft"):
        flop, elems = fft_flop, full
    elif op in ("fft-unordered", "ifft-unordered"):
        flop, elems = fft_flop, bare
    elif op == "conv-std":
        flop, elems = 2.0 * fft_flop + 6.0 * nd, 2.0 * full + 3.0 * nd
    else:  # conv-pa
        flop, elems = 2.0 * fft_flop + 6.0 * nd, 2.0 * bare + 3.0 * nd
    b = batch if op != "prepare-filter" else 1
    return flop * b, esize * elems * b


def run(op, radix, dims, batch=1, reps=5, warmup=1, seed=0x5EED5EED5EED5EED, precision="f64"):
    import numpy as np
    import torch
    import paper_2506_12718_b200 as pf

    prec = pf.F64 if precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    plan = pf.Plan(radix, dims, precision=prec)
    n = plan.total
    xs = np.stack([pf.fill_uniform(seed + b, n) for b in range(batch)])
    x0 = torch.from_numpy(xs).to("cuda", cdt)
    g = torch.from_numpy(pf.fill_uniform(seed + 1, n)).to("cuda", cdt)
    filt = pf.prepare_filter_device(g, plan)
    x = x0.clone()

    def apply():
        if op == "permute":
            pf.permute_(x, plan)
        elif op == "fft":
            pf.fft_forward_(x, plan)
        elif op == "fft-unordered":
            pf.fft_forward_unordered_(x, plan)
        elif op == "ifft":
            pf.fft_backward_(x, plan)
        elif op == "ifft-unordered":
            pf.fft_backward_unordered_(x, plan)
        elif op == "conv-std":
            pf.convolve_standard_(x, g, plan)
        elif op == "conv-pa":
            pf.convolve_permfree_(x, filt, plan)
        elif op == "prepare-filter":
            pf.prepare_filter_device(g, plan)
        else:
            raise ValueError(f"unknown op '{op}'")

    # sanity on the benchmark input before timing (bench.cpp:274-292)
    if op in ("conv-std", "conv-pa"):
        a, b = x0.clone(), x0.clone()
        pf.convolve_standard_(a, g, plan)
        pf.convolve_permfree_(b, filt, plan)
        torch.cuda.synchronize()
        err = float((a - b).abs().max()) / max(1.0, float(b.abs().max()))
        if err > (1e-11 if prec == pf.F64 else 1e-4):
            raise RuntimeError(f"convolution pipelines disagree on benchmark input ({err:.3g})")
    for _ in range(warmup):
        apply()
    torch.cuda.synchronize()
    pf.reset_permutation_pass_count()
    secs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        apply()
        e1.record()
        torch.cuda.synchronize()
        secs.append(e0.elapsed_time(e1) * 1e-3)
    passes = pf.permutation_pass_count()
    esize = 16 if prec == pf.F64 else 8
    flop, nbytes = flop_bytes(op, n, radix, batch, esize)
    med = statistics.median(secs)
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    items = (batch if op != "prepare-filter" else 1) / med
    return {"op": op, "radix": radix, "dims": "x".join(map(str, dims)), "total_n": n, "reps": reps,
            "median_s": med, "min_s": min(secs), "flop_est": flop, "bytes_est": nbytes,
            "ai_est": flop / nbytes if nbytes else 0.0, "batch": batch, "items_per_s": items,
            "model_gbs": nbytes / med / 1e9, "pct_hbm_peak": 100.0 * nbytes / med / 1e9 / peak,
            "precision": precision, "timed_permutation_passes": passes}


def emit(records, fmt="csv"):
    """bench.cpp:255-311 table, GPU columns appended."""
    cols = HEADER + GPU_COLS

    def cell(r, c):
        v = r[c]
        if c in ("median_s", "min_s", "ai_est"):
            return f"{v:.6g}"
        if c in ("flop_est", "bytes_est"):
            return f"{v:.10g}"
        if c in ("items_per_s", "model_gbs", "pct_hbm_peak"):
            return f"{v:.4g}"
        return str(v)

    rows = [[cell(r, c) for c in cols] for r in records]
    if fmt == "csv":
        return "\n".join([",".join(cols)] + [",".join(r) for r in rows]) + "\n"
    width = [max(len(c), *(len(r[i]) for r in rows)) for i, c in enumerate(cols)]
    line = lambda cells: "| " + " | ".join(x.ljust(w) for x, w in zip(cells, width)) + " |"  # noqa: E731
    return "\n".join([line(cols), "|" + "|".join("-" * (w + 2) for w in width) + "|"] + [line(r) for r in rows]) + "\n"


def main(argv=None):
    ap = argparse.ArgumentParser(prog="pafft-b200 bench")
    ap.add_argument("--op", default="conv-pa", help=f"one of {OPS} or 'all'")
    ap.add_argument("--radix", type=int, default=2)
    ap.add_argument("--dims", default="1048576")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--seed", type=lambda v: int(v, 0), default=0x5EED5EED5EED5EED)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--format", default="csv", choices=["csv", "md"])
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    if a.reps < 1 or a.warmup < 0:
        print("reps must be >= 1 and warmup >= 0", file=sys.stderr)
        return 2
    ops = OPS if a.op == "all" else [a.op]
    try:
        recs = [run(op, a.radix, parse_dims(a.dims), a.batch, a.reps, a.warmup, a.seed, a.precision) for op in ops]
    except (ValueError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    table = emit(recs, a.format)
    if a.out:
        open(a.out, "w").write(table)
    else:
        sys.stdout.write(table)
    print(f"# bench radix={a.radix} dims={a.dims} batch={a.batch} reps={a.reps} warmup={a.warmup} seed={a.seed} "
          f"prng=splitmix64 clock=cuda_events passes="
          + ",".join(f"{r['op']}:{r['timed_permutation_passes']}" for r in recs), file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
