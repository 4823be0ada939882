"""Do the HBM-bound strided pass and the FP64-bound CONV pass overlap when they
co-run on disjoint SM sets?  DIF on signals [0, B/2) and CONV on [B/2, B) (no
dependency between them), launched on two streams with persistent-grid caps.
usage: python tools/corun_probe.py [config]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2506_12718_b200 as pf
from paper_2506_12718_b200 import workload

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = workload.get_config(idx, "f64")
plan = pf.Plan(cfg.radix, cfg.dims, precision=pf.F64)
filt = pf.prepare_filter_from_impulse(torch.from_numpy(workload.impulse(cfg)).to("cuda", torch.complex128), plan)
n = int(torch.tensor(cfg.dims).prod())
B = cfg.batch
h = B // 2
x = torch.randn(B, n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nsm = torch.cuda.get_device_properties(0).multi_processor_count


def run_pass(i, lo, cnt, cap, stream):
    os.environ["PAFFT_PASS_GRID_CAP"] = str(cap)
    pf._check(pf.lib.pafft_convolve_permfree_pass(plan._h, filt._h, C.c_void_p(x[lo].data_ptr()),
                                                  C.c_void_p(y[lo].data_ptr()), cnt, i, C.c_void_p(stream.cuda_stream)))


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


td = timed(lambda: run_pass(0, 0, h, 0, s1))
tc = timed(lambda: run_pass(1, h, h, 0, s2))
print(f"config {idx}: DIF({h}) alone {td:.3f} ms, CONV({h}) alone {tc:.3f} ms, sequential sum {td + tc:.3f} ms")
for ns in (37, 50, 60, 74, 90, 110):
    def both():
        run_pass(0, 0, h, ns, s1)             # strided CTAs first (one per SM)
        run_pass(1, h, h, 3 * (nsm - ns), s2)  # CONV CTAs on the remaining SMs
    t = timed(both)
    print(f"  co-run DIF on {ns} SMs + CONV on {nsm - ns} SMs: {t:.3f} ms  ({(td + tc) / t:.2f}x vs sequential)")
