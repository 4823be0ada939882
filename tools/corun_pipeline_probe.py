"""Probe: software-pipelined passes on two streams with co-resident CTAs.
The batch is cut into chunks; the strided passes (DIF of chunk k+1, DIT of chunk
k-1) run on one stream while the CONV pass of chunk k runs on another, each
with a persistent-grid cap (PAFFT_PASS_GRID_CAP) chosen so that CTAs of both
kernels fit on every SM at once: the HBM-bound strided tiles and the FP-bound
CONV tiles then share each SM's pipes.  Timing only (random inputs).

python tools/corun_pipeline_probe.py --config 5 --precision f64 --chunks 512,256 --caps 296:148,444:148
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_12718_b200 as pf  # noqa: E402
from paper_2506_12718_b200 import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--chunks", default="512,256")
    ap.add_argument("--caps", default="296:148", help="strided:conv grid caps, comma list (0 = uncapped)")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = workload.get_config(a.config, a.precision)
    B = cfg.batch
    prec = pf.F64 if a.precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    plan = pf.Plan(cfg.radix, cfg.dims, precision=prec, device=0)
    N = cfg.total
    npass = plan.num_passes()
    assert npass == 3, "probe written for 3-pass plans"
    filt = pf.prepare_filter_from_impulse(torch.randn(N, dtype=cdt, device="cuda"), plan)
    x = torch.rand(B, N, dtype=cdt, device="cuda")
    y = torch.empty_like(x)
    sA, sC = torch.cuda.Stream(), torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    def one_pass(i, lo, cnt, cap, stream):
        os.environ["PAFFT_PASS_GRID_CAP"] = str(cap)
        pf._check(pf.lib.pafft_convolve_permfree_pass(plan._h, filt._h, C.c_void_p(x[lo].data_ptr()),
                                                      C.c_void_p(y[lo].data_ptr()), cnt, i,
                                                      C.c_void_p(stream.cuda_stream)))

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            fn()
            e1.record(main_s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    base = timed(lambda: pf.convolve_permfree_out(x, y, filt, plan, stream=main_s))
    print(f"config {a.config} {a.precision} batch {B}: one call {base:.3f} ms  {B / base * 1e3:.0f} conv/s", flush=True)
    for caps in a.caps.split(","):
        cs, cc = [int(v) for v in caps.split(":")]
        for c in [int(v) for v in a.chunks.split(",")]:
            spans = [(b0, min(B, b0 + c) - b0) for b0 in range(0, B, c)]
            K = len(spans)

            def run():
                ev0 = torch.cuda.Event()
                ev0.record(main_s)
                sA.wait_event(ev0)
                sC.wait_event(ev0)
                evD = [torch.cuda.Event() for _ in range(K)]
                evC = [torch.cuda.Event() for _ in range(K)]

                def dif(k):
                    one_pass(0, spans[k][0], spans[k][1], cs, sA)
                    evD[k].record(sA)

                def conv(k):
                    sC.wait_event(evD[k])
                    one_pass(1, spans[k][0], spans[k][1], cc, sC)
                    evC[k].record(sC)

                def dit(k):
                    sA.wait_event(evC[k])
                    one_pass(2, spans[k][0], spans[k][1], cs, sA)

                dif(0)
                for k in range(K):
                    conv(k)
                    if k + 1 < K:
                        dif(k + 1)
                    if k >= 1:
                        dit(k - 1)
                dit(K - 1)
                e = torch.cuda.Event()
                e.record(sA)
                main_s.wait_event(e)
                e2 = torch.cuda.Event()
                e2.record(sC)
                main_s.wait_event(e2)

            t = timed(run)
            print(f"  caps strided {cs} conv {cc} chunk {c:5d} ({K} chunks): {t:.3f} ms  {B / t * 1e3:.0f} conv/s  "
                  f"({base / t:.3f}x)", flush=True)
    os.environ["PAFFT_PASS_GRID_CAP"] = "0"


if __name__ == "__main__":
    main()
