"""Per-CTA retire times of each pass launch (PAFFT_PASS_TRACE=1), static and
dynamic tile order: how ragged is the tail of a persistent launch?
PAFFT_LIB=ab/libtrace.so python tools/pass_trace.py --config 5 --precision f64  (tools/trace_build.sh builds it)"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_12718_b200 as pf  # noqa: E402
from paper_2506_12718_b200 import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--precision", default="f64")
a = ap.parse_args()
cfg = workload.get_config(a.config, a.precision)
prec = pf.F64 if a.precision == "f64" else pf.F32
cdt = torch.complex128 if prec == pf.F64 else torch.complex64
plan = pf.Plan(cfg.radix, cfg.dims, precision=prec, device=0)
N, B = cfg.total, (cfg.batch if a.config != 1 else 1)
filt = pf.prepare_filter_from_impulse(torch.randn(N, dtype=cdt, device="cuda"), plan)
x = torch.rand(B, N, dtype=cdt, device="cuda")
y = torch.empty_like(x)
for dyn in (0, 4):
    os.environ["PAFFT_DYN_MIN_TILES"] = str(dyn)
    os.environ["PAFFT_PASS_TRACE"] = "0"
    for _ in range(3):
        pf.convolve_permfree_out(x, y, filt, plan)
    torch.cuda.synchronize()
    n0 = pf.dynamic_launch_count()
    os.environ["PAFFT_PASS_TRACE"] = "1"
    print(f"config {a.config} {a.precision} PAFFT_DYN_MIN_TILES={dyn}", file=sys.stderr, flush=True)
    for _ in range(2):
        pf.convolve_permfree_out(x, y, filt, plan)
    torch.cuda.synchronize()
    print(f"  dynamic launches: {pf.dynamic_launch_count() - n0}", file=sys.stderr, flush=True)
os.environ["PAFFT_PASS_TRACE"] = "0"
