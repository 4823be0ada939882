#!/usr/bin/env python
"""bench.py -- throughput of the permutation-avoiding convolution hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--precision f64|f32]
    python bench.py --impl reference ...      (the reference CPU path, same metric)

One "step" = one pass of the hot path (pafft::convolve_permfree,
convolution.cpp:45-52) over one batch of the BASELINE.json configuration:
config 2 by default (BASELINE configs[1]: n = 3^13, radix 3, batch 64, fp64).
Inputs are seeded synthetic data with BASELINE's distributions (workload.py).
Multi-GPU: one process per GPU (torchrun), batch shards with a fixed batch
per GPU (weak scaling), the prepared filter is broadcast once over NCCL,
no per-step communication; time = max over ranks of CUDA-event time.

Prints ONE JSON line (rank 0).  `value` is device-resident throughput
(inputs in HBM before timing, out-of-place so every step reads fresh inputs
larger than L2); `e2e` is the same metric through the host-buffer C-ABI call
(pinned H2D + conv + D2H inside the timed region); `roofline` is the dominant
kernel against the measured HBM peak; `cpu_baseline` is the reference CPU path
on this host's cores (oracle/_ref for radix 2/4/8, the oracle port for 3/5).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KIND_NAMES = {0: "dif", 1: "dit_fwd", 2: "dit_conj", 3: "conv_mid"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch override (0 = config batch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--graph", type=int, default=-1,
                    help="capture a step in a CUDA graph (default: on for multi-call steps, config 1)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = []
        for ts, line in self.lines:
            if t0 is not None and not (t0 <= ts <= t1):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[4:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, r in rows:
            for nm, v in zip(names, r[1:5]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


# ------------------------------------------------------------- CPU baseline
def cpu_comparator(cfg, count, threads):
    """Returns (run() -> seconds for `count` convs, kind, sample_desc).  TEST/BASELINE
    leg only: this is the one place bench.py executes oracle/ (as the timed CPU
    comparator, never as the measured product)."""
    import numpy as np
    import oracle
    from paper_2506_12718_b200 import workload

    h = workload.impulse(cfg)
    xs = workload.signals(cfg, 0, count)
    if cfg.radix in (2, 4, 8) and oracle.Ref.available():
        R = oracle.Ref()
        rp = R.plan(cfg.radix, cfg.dims)
        ghat = rp.prepare_filter(rp.filter_from_impulse(h))
        batch = rp.batch(ghat, xs)
        return (lambda: batch.run(threads)), "reference", \
            f"pafft::convolve_permfree (reference library built from its sources), {count} signals of the workload"
    O = oracle.Oracle()
    op = O.plan(cfg.radix, cfg.dims)
    ghat = op.prepare_filter(op.filter_from_impulse(h))
    gr, gi = np.ascontiguousarray(ghat.real), np.ascontiguousarray(ghat.imag)
    re0, im0 = np.ascontiguousarray(xs.real), np.ascontiguousarray(xs.imag)
    # radix 3/5 (not representable in pafft, core.hpp:14-19): pafft's ladder
    # loop nest with a hand-expanded radix-r combine (oracle/fast_ladders.c);
    # its radix-2 instance runs at pafft's own speed (tools/port_calibration.py)
    fast = len(cfg.dims) == 1 and cfg.radix in (2, 3, 4, 5)
    conv = op.convolve_permfree_fast_batch_split if fast else op.convolve_permfree_batch_split

    def run():
        re, im = re0.copy(), im0.copy()
        t = time.perf_counter()
        conv(gr, gi, re, im, count, threads)
        return time.perf_counter() - t

    what = ("pafft's ladder loop nest with a hand-expanded radix-%d combine (oracle/fast_ladders.c; its radix-2 "
            "instance matches pafft's own speed, tools/port_calibration.py)" % cfg.radix) if fast else \
        "oracle restatement of pafft's ladders"
    return run, "port", f"{what}; radix {cfg.radix} is not representable in pafft (core.hpp:14-19); " \
                        f"{count} signals of the workload"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample_count(cfg, threads):
    # bounded: ~10-30 s of CPU work at ~20 ns per point-stage per core
    work_per_conv = cfg.total * sum(cfg.stages) * 2 * 2e-8  # seconds per conv per core, rough
    count = max(threads, int(round(20.0 / max(work_per_conv, 1e-6))))
    return max(1, min(count, threads * 4, cfg.batch * cfg.calls))


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    threads = cpu_threads()
    count = cpu_sample_count(cfg, threads)
    run, kind, sample = cpu_comparator(cfg, count, threads)
    for _ in range(min(args.warmup, 1)):
        run()
    secs = [run() for _ in range(args.steps)]
    total = sum(secs)
    value = count * len(secs) / total
    line = {
        "impl": "reference", "metric": "convolutions_per_second", "value": value, "unit": "conv/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(secs), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, BASELINE distributions)",
        "config": {"workload": f"config{cfg.idx}: {cfg.note}", "radix": cfg.radix, "dims": cfg.dims,
                   "batch_per_step": count, "precision": "f64"},
        "cpu_baseline": {"value": value, "unit": "conv/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "conv/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def main():
    args = parse()
    from paper_2506_12718_b200 import workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = workload.get_config(args.config, args.precision)

    if args.impl == "reference":
        run_reference(args, workload.get_config(args.config, "f64"), rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2506_12718_b200 as pf

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    prec = pf.F64 if cfg.precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    ndt = np.complex128 if prec == pf.F64 else np.complex64
    plan = pf.Plan(cfg.radix, cfg.dims, precision=prec, device=local)
    N = cfg.total
    S = workload.signal_bytes(cfg)

    # ---- prepared filter: rank 0 prepares, one NCCL broadcast over NVLink
    t_prep = time.perf_counter()
    if rank == 0:
        h = torch.from_numpy(workload.impulse(cfg).astype(ndt)).to(dev)
        filt = pf.prepare_filter_from_impulse(h, plan)
        del h
    else:
        filt = pf.empty_filter(plan)
    if world > 1:
        from paper_2506_12718_b200 import dist as pdist
        pdist.broadcast_filter_tensors([pf.filter_device_tensor(filt), pf.filter_device_tensor(filt, scaled=True)])
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t_prep

    # ---- inputs: per-rank shard (fixed per-GPU batch), resident in HBM
    from paper_2506_12718_b200 import dist as pdist
    per = args.batch or (cfg.calls if cfg.calls > 1 else cfg.batch)
    first, per = pdist.shard(per, rank)
    host = torch.empty((per, N), dtype=cdt, pin_memory=True)
    hv = host.numpy()
    if prec == pf.F64:
        workload.signals(cfg, first, per, out=hv)
    else:
        hv[:] = workload.signals(cfg, first, per).astype(np.complex64)
    x = host.to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    npass = plan.num_passes()
    infos = []
    import ctypes as C
    for i in range(npass):
        k, a, R, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        pf._check(pf.lib.pafft_plan_pass_info(plan._h, i, C.byref(k), C.byref(a), C.byref(R), C.byref(s)))
        infos.append({"kind": KIND_NAMES[k.value], "axis": a.value, "R": R.value, "stages": s.value})

    calls = cfg.calls if cfg.calls > 1 else 1
    bpc = per // calls  # signals per call
    sptr = C.c_void_p(stream.cuda_stream)
    chunk = int(pf.lib.pafft_plan_chunk_signals(plan._h)) or bpc
    chunk = max(1, min(chunk, bpc))
    esz = x.element_size()

    def launch_pass(i, xs, ys, nb):
        pf._check(pf.lib.pafft_convolve_permfree_pass(plan._h, filt._h, C.c_void_p(xs), C.c_void_p(ys), nb, i, sptr))

    def step():
        # the public hot-path call: convolve_permfree out of place, per call
        for c in range(calls):
            xs = x.data_ptr() + c * bpc * N * esz
            ys = y.data_ptr() + c * bpc * N * esz
            pf._check(pf.lib.pafft_convolve_permfree_oop(plan._h, filt._h, C.c_void_p(xs), C.c_void_p(ys), bpc,
                                                         sptr))

    gpu_index = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        try:
            gpu_index = int(cvd.split(",")[local])
        except ValueError:
            pass
    sampler = ClockSampler(gpu_index)
    sampler.start()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # launch-bound multi-call steps (config 1: 100 batch-1 calls) replay a
    # captured CUDA graph of the same calls instead of re-launching from Python
    use_graph = args.graph if args.graph >= 0 else int(calls > 1)
    graph_launches = 0
    if use_graph:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        l0 = pf.kernel_launch_count()
        with torch.cuda.stream(cs):
            sptr_saved = sptr
            sptr = C.c_void_p(cs.cuda_stream)
            with torch.cuda.graph(g, stream=cs):
                step()
            sptr = sptr_saved
        graph_launches = pf.kernel_launch_count() - l0
        stream.wait_stream(cs)
        plain_step = step

        def step():  # noqa: F811
            g.replay()

        step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region (device-resident, CUDA events, max over ranks)
    launches0 = pf.kernel_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tw0 = time.time()
    e0.record(stream)
    for k in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    if world > 1:
        dist.barrier()
    launches = pf.kernel_launch_count() - launches0 + graph_launches * args.steps
    ms_max = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    # keep the GPU busy (untimed) until the clock sampler has >= 1 s of samples
    t_soak = time.time()
    while time.time() - tw0 < 1.2 and time.time() - t_soak < 3.0:
        step()
        torch.cuda.synchronize()
    tw_end = time.time()
    sampler.stop()
    clocks = sampler.summary(tw0 - 0.05, tw_end + 0.05)

    # ---- per-pass device time: the same launches the pipeline issues (one
    # L2 chunk per launch), run one at a time on one stream between CUDA events
    reps = max(1, min(args.steps, 8))
    nch = max(1, bpc // chunk)
    pev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(npass)]
           for _ in range(reps * nch)]
    for r in range(reps):
        for q in range(nch):
            xs = x.data_ptr() + q * chunk * N * esz
            ys = y.data_ptr() + q * chunk * N * esz
            for i in range(npass):
                ev = pev[r * nch + q][i]
                ev[0].record(stream)
                launch_pass(i, xs, ys, chunk)
                ev[1].record(stream)
    torch.cuda.synchronize()
    pass_ms = [statistics.mean(ev[i][0].elapsed_time(ev[i][1]) for ev in pev) for i in range(npass)]
    dom = max(range(npass), key=lambda i: pass_ms[i])
    dom_bytes = 2.0 * S * chunk + (S if infos[dom]["kind"] == "conv_mid" else 0.0)
    peak, peak_src = measured_peak()
    achieved = dom_bytes / (pass_ms[dom] * 1e-3) / 1e9

    convs = per * world * args.steps
    value = convs / (ms_max * 1e-3)
    conv_gbs = value / world * workload.bytes_per_conv(cfg, world) / 1e9
    flops = workload.flops_per_conv(cfg)
    fp_peak = 34.08 if cfg.precision == "f64" else 72.06  # DFMA / FFMA TFLOP/s, measured

    # ---- e2e: host buffers through the C-ABI (pinned H2D + conv + D2H timed)
    e2e = None
    if not args.no_e2e:
        yh = torch.empty_like(host, pin_memory=True)
        ysteps = args.e2e_steps or max(2, min(args.steps, 5))
        xv, yv = host.numpy(), yh.numpy()

        def host_step():
            for c in range(calls):
                xs = xv[c * bpc:(c + 1) * bpc]
                ys = yv[c * bpc:(c + 1) * bpc]
                pf._check(pf.lib.pafft_convolve_permfree_host_oop(plan._h, filt._h, C.c_void_p(xs.ctypes.data),
                                                                  C.c_void_p(ys.ctypes.data), bpc))

        host_step()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(ysteps):
            host_step()
        et = pdist.max_over_ranks(time.perf_counter() - t, dev)
        e2e = {"value": per * world * ysteps / et, "unit": "conv/s", "h2d_bytes_per_step": per * S,
               "d2h_bytes_per_step": per * S, "steps": ysteps, "pipelined": "3 streams, 64 MiB chunks, pinned"}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            c64 = workload.get_config(args.config, "f64")
            threads = cpu_threads()
            count = cpu_sample_count(c64, threads)
            run, kind, sample = cpu_comparator(c64, count, threads)
            secs = run()
            # one core, pafft's own methodology (bench.cpp:52-59)
            run1, _, _ = cpu_comparator(c64, 1, 1)
            secs1 = run1()
            cpu = {"value": count / secs, "unit": "conv/s", "cores": threads, "kind": kind,
                   "sample": sample + f"; {threads} threads, one timed batch of {count}",
                   "value_1core": 1.0 / secs1}
        except Exception as e:  # report, never substitute
            cpu = {"value": None, "unit": "conv/s", "cores": cpu_threads(), "kind": "unavailable",
                   "sample": f"{type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": "convolutions_per_second",
            "value": value,
            "unit": "conv/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": cfg.precision,
            "data": "synthetic (seeded SplitMix64, BASELINE distributions; inputs device-resident, out of place)",
            "config": {"workload": f"config{cfg.idx}: {cfg.note}", "radix": cfg.radix, "dims": cfg.dims,
                       "batch_per_gpu": per, "calls_per_step": calls, "global_batch": per * world,
                       "precision": cfg.precision, "parallelism": f"batch-sharded x{world}",
                       "cuda_graph": bool(use_graph),
                       "l2": f"inputs {per * S / 2**30:.2f} GiB per GPU per step > 126 MB L2 (no flush needed)"
                       if per * S > 2 * 126e6 else "inputs smaller than 2x L2; out-of-place fresh buffer per call"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(f"config{cfg.idx}_{cfg.precision}"),
                         "kernel": f"pass{dom}:{infos[dom]['kind']}(R={infos[dom]['R']})",
                         "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": pass_ms[dom],
                         "signals_per_launch": chunk,
                         "peak_source": peak_src,
                         # what binds it (ncu --set full of the same kernel, committed)
                         "ncu_pipes": ncu_traffic(f"config{cfg.idx}_{cfg.precision}_pipes")},
            "conv_roofline": {"bytes_per_conv": workload.bytes_per_conv(cfg, world), "achieved_gbs_per_gpu": conv_gbs,
                              "frac_of_hbm": conv_gbs / peak, "frac_of_hbm_datasheet_8tbs": conv_gbs / 8000.0,
                              "flops_per_conv": flops, "achieved_tflops_per_gpu": value / world * flops / 1e12,
                              # FP peaks measured by tools/probes/peaks.cu (profiles/r01_peaks_probe.log)
                              "fp_peak_tflops": fp_peak, "frac_of_fp_peak": value / world * flops / 1e12 / fp_peak},
            "passes": [{**infos[i], "ms": pass_ms[i]} for i in range(npass)],
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "prepare_filter_s": t_prep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
