#!/usr/bin/env python
"""bench.py -- throughput of the permutation-avoiding convolution hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--precision f64|f32]
    python bench.py --impl reference ...      (the reference CPU path, same metric)

One "step" = one pass of the hot path (pafft::convolve_permfree,
convolution.cpp:45-52) over one batch of the BASELINE.json configuration:
config 2 by default (BASELINE configs[1]: n = 3^13, radix 3, batch 64, fp64).
Inputs are seeded synthetic data with BASELINE's distributions (workload.py).

Multi-GPU: one process per GPU (torchrun).  The config's FIXED
global batch is split into contiguous slices, batch / G per rank (strong
scaling; `--weak` keeps a fixed per-GPU batch instead); config 1's 100-call
sequence runs as replicas.  The prepared filter is broadcast once over NCCL,
there is no per-step communication; time = max over ranks of CUDA-event time.

Prints ONE JSON line (rank 0).  `value` is device-resident throughput
(inputs in HBM before timing, out-of-place so every step reads fresh inputs
larger than L2); `e2e` is the same metric through the host-buffer C-ABI call
(pinned H2D + conv + D2H inside the timed region); `roofline` is the dominant
kernel against the measured HBM peak; `cpu_baseline` is the reference CPU path
on this host's cores (oracle/_ref = pafft itself for radix 2/4/8, the
pafft-style port for 3/5), 1 warm-up + 3 timed repetitions, median.  With the
default config the line also carries `configs`: the same measurement for
every other BASELINE config (1, 3, 4, 5 fp64, 5 fp32) at fewer steps.

The reference arm (`--impl reference`) never imports the product package: its
inputs come from the oracle's SplitMix64 generator (byte-identical to the
product's, tests/test_abi.py), and it times the FULL config batch per step.
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
SUB_CONFIGS = [(1, "f64"), (3, "f64"), (4, "f64"), (5, "f64"), (5, "f32"), (2, "f32")]
# measured FP peaks (tools/probes/peaks.cu, profiles/r01_peaks_probe.log): DFMA / FFMA TFLOP/s
FP_PEAK = {"f64": 34.08, "f32": 72.06}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--batch", type=int, default=0, help="global batch override (0 = config batch)")
    ap.add_argument("--weak", action="store_true", help="fixed per-GPU batch (weak scaling) instead of a split")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the per-config sub-results")
    ap.add_argument("--sub-steps", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--graph", type=int, default=-1,
                    help="capture a step in a CUDA graph (default: on for multi-call steps, config 1)")
    return ap.parse_args()


def workload_mod():
    """workload.py loaded by path as a standalone module: importing it through
    the package would run paper_2506_12718_b200/__init__.py, which maps the
    product library -- the reference arm must never do that."""
    mod = sys.modules.get("_pafft_workload")
    if mod is None:
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "_pafft_workload", os.path.join(ROOT, "paper_2506_12718_b200", "workload.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules["_pafft_workload"] = mod
        spec.loader.exec_module(mod)
    return mod


def repo_libs_loaded():
    """Shared objects under the repo this process has mapped (/proc/self/maps):
    the reference arm must show only oracle/*, the GPU arm the product library."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(ROOT)):
                    libs.add(os.path.relpath(os.path.realpath(path), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(libs)


def cfg_key(idx, prec):
    return f"config{idx}" + ("" if prec == "f64" else "_" + prec)


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


def ncu_info(key):
    """Per-launch figures of a config's dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


# ------------------------------------------------------------- CPU baseline
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuComparator:
    """The reference CPU path on this host (TEST/BASELINE leg only: the one place
    bench.py executes oracle/, as the timed comparator, never as the product).
    radix 2/4/8: pafft::convolve_permfree itself (oracle/_ref, compiled from the
    reference's sources); radix 3/5 (not representable in pafft, core.hpp:14-19):
    pafft's ladder loop nest with a hand-expanded radix-r combine
    (oracle/fast_ladders.c; its radix-2 instance runs at pafft's own speed,
    profiles/r01_cpu_port_calibration.log).  Inputs from the oracle's SplitMix64
    (identical bytes to the product generator); this process never maps the
    product library."""

    def __init__(self, cfg, count):
        import numpy as np
        import oracle
        workload = workload_mod()

        self.cfg, self.count = cfg, count
        O = oracle.Oracle()
        h = workload.impulse(cfg, fill_normal=O.fill_normal)
        seeds = [workload.seed_signal(b) for b in range(count)]
        self.re0, self.im0 = O.fill_signals_split(cfg.signal == "uniform", seeds, cfg.total)
        self.ref = cfg.radix in (2, 4, 8) and oracle.Ref.available()
        if self.ref:
            R = oracle.Ref()
            self.rp = R.plan(cfg.radix, cfg.dims)
            self.ghat = self.rp.prepare_filter(self.rp.filter_from_impulse(h))
            self.kind = "reference"
            self.what = "pafft::convolve_permfree (the reference library built from its own sources, oracle/_ref)"
        else:
            op = O.plan(cfg.radix, cfg.dims)
            self.op = op
            ghat = op.prepare_filter(op.filter_from_impulse(h))
            self.gr, self.gi = np.ascontiguousarray(ghat.real), np.ascontiguousarray(ghat.imag)
            fast = len(cfg.dims) == 1 and cfg.radix in (2, 3, 4, 5)
            self.conv = op.convolve_permfree_fast_batch_split if fast else op.convolve_permfree_batch_split
            self.kind = "port"
            self.what = (f"pafft's ladder loop nest with a hand-expanded radix-{cfg.radix} combine "
                         "(oracle/fast_ladders.c); radix %d is not representable in pafft (core.hpp:14-19)"
                         % cfg.radix) if fast else "oracle restatement of pafft's ladders"

    def run(self, threads, count=None):
        """Seconds for one batch of `count` convolutions (inputs re-staged
        outside the timed region, so every repetition convolves fresh signals)."""
        n = count or self.count
        if self.ref:
            batch = self.rp.batch_split(self.ghat, self.re0[:n], self.im0[:n])
            return batch.run(threads)
        re, im = self.re0[:n].copy(), self.im0[:n].copy()
        t = time.perf_counter()
        self.conv(self.gr, self.gi, re, im, n, threads)
        return time.perf_counter() - t


def pinned_one_core(fn):
    """Run fn() with this thread (and the threads it spawns) pinned to one core,
    pafft's methodology (bench.cpp:52-59)."""
    try:
        old = os.sched_getaffinity(0)
    except AttributeError:
        return fn(), None
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        return fn(), core
    finally:
        os.sched_setaffinity(0, old)


def cpu_measure(cfg, count, reps=3, warmup=1, one_core=True):
    """1 warm-up, >= 3 repetitions, median; all host cores sharing
    one plan/filter over the batch, plus one pinned core."""
    threads = cpu_threads()
    comp = CpuComparator(cfg, count)
    for _ in range(warmup):
        comp.run(threads)
    secs = [comp.run(threads) for _ in range(reps)]
    med = statistics.median(secs)
    out = {"value": count / med, "unit": "conv/s", "cores": threads, "kind": comp.kind,
           "sample": f"{comp.what}; {count} signals of the workload per repetition, {threads} threads sharing one "
                     f"plan and prepared filter; {warmup} warm-up + {reps} repetitions, median",
           "reps_s": secs}
    if one_core:
        def one():
            comp.run(1, 1)
            return statistics.median([comp.run(1, 1) for _ in range(reps)])
        s1, core = pinned_one_core(one)
        out["value_1core"] = 1.0 / s1
        out["one_core"] = f"1 signal per repetition, pinned to cpu {core}, {warmup} warm-up + {reps} reps, median"
    return out


def run_reference(args, rank):
    """`--impl reference`: the reference CPU path on all host cores, the full
    config batch per step (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    workload = workload_mod()

    def measure(cfg, steps, warmup):
        count = cfg.calls if cfg.calls > 1 else cfg.batch
        comp = CpuComparator(cfg, count)
        threads = cpu_threads()
        for _ in range(warmup):
            comp.run(threads)
        secs = [comp.run(threads) for _ in range(steps)]
        return comp, threads, count, secs

    cfg = workload.get_config(args.config, "f64")
    comp, threads, count, secs = measure(cfg, args.steps, args.warmup)
    total = sum(secs)
    value = count * len(secs) / total
    line = {
        "impl": "reference", "metric": "convolutions_per_second", "value": value, "unit": "conv/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(secs), "higher_is_better": True,
        "scaling": "weak" if cfg.calls > 1 or args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, BASELINE distributions)",
        "config": {"workload": f"config{cfg.idx}: {cfg.note}", "radix": cfg.radix, "dims": cfg.dims,
                   "global_batch": count, "batch_per_step": count, "precision": "f64"},
        "cpu_baseline": {"value": value, "unit": "conv/s", "cores": threads, "kind": comp.kind,
                         "sample": f"{comp.what}; the full batch of {count} signals per step, {threads} threads"},
        "e2e": {"value": value, "unit": "conv/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s": {"median": statistics.median(secs), "min": min(secs), "max": max(secs)},
    }
    if not args.no_sub and args.config == 2:
        subs = {}
        for idx, prec in SUB_CONFIGS:
            if prec != "f64":
                subs[cfg_key(idx, prec)] = {"same_as": cfg_key(idx, "f64"),
                                            "note": "no fp32 CPU path: the fp32 GPU result is checked against the "
                                                    "fp64 pipeline on rounded inputs (BASELINE.md 4)"}
                continue
            c = workload.get_config(idx, "f64")
            k = max(3, min(args.sub_steps, 3))
            comp, threads, count, secs = measure(c, k, 1)
            med = statistics.median(secs)
            subs[cfg_key(idx, prec)] = {"value": count / med, "unit": "conv/s", "cores": threads, "kind": comp.kind,
                                        "batch_per_step": count, "steps": k, "warmup": 1,
                                        "step_s_median": med, "workload": f"config{idx}: {c.note}"}
            del comp
        line["configs"] = subs
    line["repo_libs_loaded"] = repo_libs_loaded()
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
class Gpu:
    """Per-process GPU context (device, rank, world, process group)."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # PAFFT_BENCH_BACKEND=gloo: a plumbing check of the multi-rank flow
        # (partition, filter broadcast, max over ranks, rank-0 line) with ranks
        # that may share a GPU (device = local rank mod device count); its
        # timings are not a measurement.  Default: NCCL, one GPU per rank.
        backend = os.environ.get("PAFFT_BENCH_BACKEND", "nccl")
        self.device_index = self.local % max(1, torch.cuda.device_count()) if backend != "nccl" else self.local
        torch.cuda.set_device(self.device_index)
        if self.world > 1:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device_index))
            else:
                dist.init_process_group(backend)
        self.dev = torch.device("cuda", self.device_index)
        self.local = self.device_index
        self.gpu_index = self.local
        cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
        if cvd:
            try:
                self.gpu_index = int(cvd.split(",")[self.local])
            except ValueError:
                pass

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()


def gpu_measure(g, cfg, args, steps, warmup, with_e2e, with_cpu):
    """One BASELINE config through the product path on this rank's shard."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2506_12718_b200 as pf
    from paper_2506_12718_b200 import dist as pdist
    from paper_2506_12718_b200 import workload

    world, rank, dev = g.world, g.rank, g.dev
    prec = pf.F64 if cfg.precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    ndt = np.complex128 if prec == pf.F64 else np.complex64
    plan = pf.Plan(cfg.radix, cfg.dims, precision=prec, device=g.local)
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
        pdist.broadcast_filter_tensors([pf.filter_device_tensor(filt), pf.filter_device_tensor(filt, scaled=True)])
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t_prep

    # ---- inputs: this rank's slice of the global batch, resident in HBM
    calls = cfg.calls if cfg.calls > 1 else 1
    weak = args.weak or calls > 1  # config 1 (the call sequence) runs as replicas
    if calls > 1:
        first, per = 0, calls
        global_batch = calls * world
    elif weak:
        per_rank = args.batch or cfg.batch
        first, per = pdist.shard_weak(per_rank, rank)
        global_batch = per_rank * world
    else:
        global_batch = args.batch or cfg.batch
        first, per = pdist.shard(global_batch, world, rank)
    host = torch.empty((max(per, 1), N), dtype=cdt, pin_memory=True)
    hv = host.numpy()
    if per:
        if prec == pf.F64:
            workload.signals(cfg, first, per, out=hv)
        else:
            for c0 in range(0, per, 256):
                c1 = min(per, c0 + 256)
                hv[c0:c1] = workload.signals(cfg, first + c0, c1 - c0).astype(np.complex64)
    x = host.to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    npass = plan.num_passes()
    infos = []
    for i in range(npass):
        k, a, R, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        pf._check(pf.lib.pafft_plan_pass_info(plan._h, i, C.byref(k), C.byref(a), C.byref(R), C.byref(s)))
        infos.append({"kind": KIND_NAMES[k.value], "axis": a.value, "R": R.value, "stages": s.value})

    bpc = per // calls  # signals per call
    sptr = [C.c_void_p(stream.cuda_stream)]
    esz = x.element_size()

    def launch_pass(i, xs, ys, nb):
        pf._check(pf.lib.pafft_convolve_permfree_pass(plan._h, filt._h, C.c_void_p(xs), C.c_void_p(ys), nb, i,
                                                      sptr[0]))

    def step():
        # the public hot-path call: convolve_permfree out of place, per call
        for c in range(calls):
            xs = x.data_ptr() + c * bpc * N * esz
            ys = y.data_ptr() + c * bpc * N * esz
            pf._check(pf.lib.pafft_convolve_permfree_oop(plan._h, filt._h, C.c_void_p(xs), C.c_void_p(ys), bpc,
                                                         sptr[0]))

    sampler = ClockSampler(g.gpu_index)
    sampler.start()
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # launch-bound multi-call steps (config 1: 100 batch-1 calls) replay a
    # captured CUDA graph of the same calls instead of re-launching from Python
    use_graph = args.graph if args.graph >= 0 else int(calls > 1)
    graph_launches = 0
    if use_graph and per:
        gr = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        l0 = pf.kernel_launch_count()
        with torch.cuda.stream(cs):
            saved = sptr[0]
            sptr[0] = C.c_void_p(cs.cuda_stream)
            with torch.cuda.graph(gr, stream=cs):
                step()
            sptr[0] = saved
        graph_launches = pf.kernel_launch_count() - l0
        stream.wait_stream(cs)

        def step():  # noqa: F811
            gr.replay()

        step()
        torch.cuda.synchronize()
    g.barrier()

    # ---- timed region (device-resident, CUDA events, max over ranks)
    launches0 = pf.kernel_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    g.barrier()
    tw0 = time.time()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    g.barrier()
    launches = pf.kernel_launch_count() - launches0 + graph_launches * steps
    ms_max = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    # keep the GPU busy (untimed) until the clock sampler has >= 1 s of samples
    t_soak = time.time()
    while time.time() - tw0 < 1.2 and time.time() - t_soak < 3.0:
        step()
        torch.cuda.synchronize()
    tw_end = time.time()
    sampler.stop()
    clocks = sampler.summary(tw0 - 0.05, tw_end + 0.05)

    # ---- config 1 only, reported beside the measurement: the same independent
    # batch-1 calls issued alternately on two streams, so consecutive calls may
    # overlap (the reference arm runs its 100 signals on all host threads at
    # once); `value` above stays the one-stream call sequence
    concurrent = None
    if calls > 1 and bpc:
        gr2 = torch.cuda.CUDAGraph()
        c1s, c2s = torch.cuda.Stream(), torch.cuda.Stream()
        c1s.wait_stream(stream)
        with torch.cuda.stream(c1s):
            with torch.cuda.graph(gr2, stream=c1s):
                c2s.wait_stream(c1s)
                for c in range(calls):
                    st = c1s if c % 2 == 0 else c2s
                    xs = x.data_ptr() + c * bpc * N * esz
                    ys = y.data_ptr() + c * bpc * N * esz
                    pf._check(pf.lib.pafft_convolve_permfree_oop(plan._h, filt._h, C.c_void_p(xs), C.c_void_p(ys),
                                                                 bpc, C.c_void_p(st.cuda_stream)))
                c1s.wait_stream(c2s)
        stream.wait_stream(c1s)
        gr2.replay()
        torch.cuda.synchronize()
        g.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(steps):
            gr2.replay()
        f1.record(stream)
        torch.cuda.synchronize()
        ms2 = pdist.max_over_ranks(f0.elapsed_time(f1), dev)
        concurrent = {"value": global_batch * steps / (ms2 * 1e-3), "unit": "conv/s", "streams": 2,
                      "note": "the same independent batch-1 calls, even calls on one stream and odd calls on "
                              "another (consecutive calls may overlap); not the headline value"}

    # ---- per-pass device time: the same launches one call issues, one at a
    # time on one stream between CUDA events
    reps = max(1, min(steps, 8))
    pass_ms = [0.0] * npass
    if bpc:
        pev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(npass)]
               for _ in range(reps)]
        for r in range(reps):
            for i in range(npass):
                ev = pev[r][i]
                ev[0].record(stream)
                launch_pass(i, x.data_ptr(), y.data_ptr(), bpc)
                ev[1].record(stream)
        torch.cuda.synchronize()
        pass_ms = [statistics.mean(ev[i][0].elapsed_time(ev[i][1]) for ev in pev) for i in range(npass)]
    dom = max(range(npass), key=lambda i: pass_ms[i])
    dom_bytes = 2.0 * S * bpc + (S if infos[dom]["kind"] == "conv_mid" else 0.0)
    peak, peak_src = measured_peak()
    achieved = dom_bytes / (pass_ms[dom] * 1e-3) / 1e9 if pass_ms[dom] > 0 else 0.0

    convs = global_batch * steps
    value = convs / (ms_max * 1e-3)
    bpc_alg = workload.bytes_per_conv(cfg, world, weak)
    conv_gbs = value / world * bpc_alg / 1e9
    flops = workload.flops_per_conv(cfg)
    fp_peak = FP_PEAK[cfg.precision]
    key = cfg_key(cfg.idx, cfg.precision)
    ncu = ncu_info(key) or {}

    # ---- e2e: host buffers through the C-ABI (pinned H2D + conv + D2H timed)
    e2e = None
    if with_e2e:
        yh = torch.empty_like(host, pin_memory=True)
        ysteps = args.e2e_steps or max(2, min(steps, 5))
        xv, yv = host.numpy(), yh.numpy()

        def host_step():
            for c in range(calls):
                xs = xv[c * bpc:(c + 1) * bpc]
                ys = yv[c * bpc:(c + 1) * bpc]
                pf._check(pf.lib.pafft_convolve_permfree_host_oop(plan._h, filt._h, C.c_void_p(xs.ctypes.data),
                                                                  C.c_void_p(ys.ctypes.data), bpc))

        host_step()
        g.barrier()
        t = time.perf_counter()
        step_ms = []
        for _ in range(ysteps):
            t1 = time.perf_counter()
            host_step()  # synchronous: returns when the results are in the host buffer
            step_ms.append(1e3 * (time.perf_counter() - t1))
        et = pdist.max_over_ranks(time.perf_counter() - t, dev)
        # value = all timed steps (mean); the per-step times show how steady the host link was
        e2e = {"value": global_batch * ysteps / et, "unit": "conv/s", "h2d_bytes_per_step": per * S,
               "d2h_bytes_per_step": per * S, "steps": ysteps, "step_ms": [round(v, 3) for v in step_ms],
               "pipelined": "3 streams, 64 MiB chunks, pinned host buffers"}
        del yh

    # ---- CPU baseline (rank 0, N = 1 only): bounded sample, median of reps
    cpu = None
    if with_cpu and rank == 0 and world == 1:
        try:
            # the whole config batch (0.5-2 s per repetition on the box's host)
            c64 = workload.get_config(cfg.idx, "f64")
            cpu = cpu_measure(c64, c64.calls if c64.calls > 1 else c64.batch)
        except Exception as e:  # report, never substitute
            cpu = {"value": None, "unit": "conv/s", "cores": cpu_threads(), "kind": "unavailable",
                   "sample": f"{type(e).__name__}: {e}"}

    out = {
        "value": value, "unit": "conv/s", "ms_per_step": ms_max / steps, "steps": steps, "warmup": warmup,
        "dtype": cfg.precision,
        "config": {"workload": f"config{cfg.idx}: {cfg.note}", "radix": cfg.radix, "dims": cfg.dims,
                   "global_batch": global_batch, "batch_per_gpu": per, "calls_per_step": calls,
                   "precision": cfg.precision,
                   "parallelism": (f"replicas x{world}" if calls > 1 else
                                   f"batch split {global_batch}/{world}" if not weak else f"weak x{world}"),
                   "cuda_graph": bool(use_graph),
                   "l2": f"inputs {per * S / 2**30:.2f} GiB per GPU per step > 126 MB L2 (no flush needed)"
                   if per * S > 2 * 126e6 else "inputs smaller than 2x L2; out-of-place fresh buffer per call"},
        "scaling": "weak" if weak else "strong",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu.get("traffic") if isinstance(ncu, dict) else None,
                     "kernel": f"pass{dom}:{infos[dom]['kind']}(R={infos[dom]['R']})",
                     "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": pass_ms[dom],
                     "signals_per_launch": bpc, "peak_source": peak_src,
                     # what actually limits that kernel (ncu --set full of the same kernel, committed)
                     "limiter": ncu.get("limiter") if isinstance(ncu, dict) else None},
        "conv_roofline": {"bytes_per_conv": bpc_alg, "achieved_gbs_per_gpu": conv_gbs,
                          "frac_of_hbm": conv_gbs / peak, "frac_of_hbm_datasheet_8tbs": conv_gbs / 8000.0,
                          "flops_per_conv": flops, "achieved_tflops_per_gpu": value / world * flops / 1e12,
                          "fp_peak_tflops": fp_peak, "frac_of_fp_peak": value / world * flops / 1e12 / fp_peak},
        "passes": [{**infos[i], "ms": pass_ms[i]} for i in range(npass)],
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "prepare_filter_s": t_prep,
    }
    if concurrent:
        out["calls_on_two_streams"] = concurrent
    del x, y, host, filt, plan
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    from paper_2506_12718_b200 import workload

    g = Gpu(args)
    cfg = workload.get_config(args.config, args.precision)
    res = gpu_measure(g, cfg, args, args.steps, args.warmup, not args.no_e2e, not args.no_cpu)
    subs = None
    if not args.no_sub and args.config == 2 and args.precision == "f64" and not args.batch:
        subs = {}
        for idx, prec in SUB_CONFIGS:
            c = workload.get_config(idx, prec)
            k = max(3, args.sub_steps)
            try:
                r = gpu_measure(g, c, args, k, 3, not args.no_e2e, False)
                subs[cfg_key(idx, prec)] = {kk: r[kk] for kk in ("value", "unit", "ms_per_step", "steps", "warmup",
                                                                 "dtype", "config", "scaling", "roofline",
                                                                 "conv_roofline", "passes", "e2e", "gpu_launches",
                                                                 "clocks", "calls_on_two_streams") if kk in r}
            except Exception as e:  # report, never substitute
                subs[cfg_key(idx, prec)] = {"error": f"{type(e).__name__}: {e}"}
    if g.rank == 0:
        line = {
            "metric": "convolutions_per_second",
            "value": res["value"],
            "unit": "conv/s",
            "n_gpus": g.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"],
            "higher_is_better": True,
            "scaling": res["scaling"],
            "vs_baseline": None,
            "dtype": res["dtype"],
            "data": "synthetic (seeded SplitMix64, BASELINE distributions; inputs device-resident, out of place)",
            **{k: res[k] for k in ("config", "roofline", "conv_roofline", "passes", "e2e", "gpu_launches", "clocks",
                                   "cpu_baseline", "prepare_filter_s", "calls_on_two_streams") if k in res},
        }
        if subs is not None:
            line["configs"] = subs
            line["gpu_launches_all_configs"] = res["gpu_launches"] + sum(
                s.get("gpu_launches", 0) for s in subs.values())
        line["repo_libs_loaded"] = repo_libs_loaded()
        print(json.dumps(line), flush=True)
    if g.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
