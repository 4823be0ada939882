"""Probe: run a config's full batch as back-to-back chunks of c signals (all
three passes per chunk before the next chunk starts) and time the whole batch.
When a chunk's intermediate (c x signal bytes) plus the prepared filter fit in
L2, the DIF pass's stores, the CONV pass's read-modify-write and the DIT pass's
loads can hit L2 instead of HBM.  Random inputs (timing only, no parity).

python tools/l2_chunk_probe.py --config 2 --chunks 64,32,16,8,4,3,2,1
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_12718_b200 as pf  # noqa: E402
from paper_2506_12718_b200 import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--chunks", default="64,32,16,8,4,3,2,1")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--streams", default="1", help="comma list: chunks are issued round-robin on this many streams")
    a = ap.parse_args()
    cfg = workload.get_config(a.config, a.precision)
    B = a.batch or cfg.batch
    prec = pf.F64 if a.precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    plan = pf.Plan(cfg.radix, cfg.dims, precision=prec, device=0)
    N = cfg.total
    h = torch.randn(N, dtype=cdt, device="cuda")
    filt = pf.prepare_filter_from_impulse(h, plan)
    x = torch.rand(B, N, dtype=cdt, device="cuda")
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    print(f"config {a.config} {a.precision} batch {B} signal {N * x.element_size() / 2**20:.1f} MiB", flush=True)
    side = [torch.cuda.Stream() for _ in range(8)]
    for c, ns in [(int(v), int(w)) for w in a.streams.split(",") for v in a.chunks.split(",")]:
        def run():
            s = torch.cuda.current_stream()  # the capture stream under --graph
            if ns > 1:
                ev = torch.cuda.Event()
                ev.record(s)
                for q in side[:ns]:
                    q.wait_event(ev)
            for i, b0 in enumerate(range(0, B, c)):
                b1 = min(B, b0 + c)
                q = s if ns == 1 else side[i % ns]
                pf.convolve_permfree_out(x[b0:b1], y[b0:b1], filt, plan, stream=q)
            if ns > 1:
                for q in side[:ns]:
                    e = torch.cuda.Event()
                    e.record(q)
                    s.wait_event(e)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        fn = run
        if a.graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run()
            fn = g.replay
            fn()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(torch.cuda.current_stream())
            fn()
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        print(f"streams {ns} chunk {c:5d}: {ms:8.3f} ms per {B} convs  {B / ms * 1e3:10.1f} conv/s  "
              f"(chunk working set {c * N * x.element_size() / 2**20:.0f} MiB + filter)", flush=True)


if __name__ == "__main__":
    main()
