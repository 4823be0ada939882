"""Time each pass alone through the fused kernel (PAFFT_FUSED_ONLY) next to the
three-launch path's per-pass times.  usage: python tools/fused_only.py config"""
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
x = torch.randn(cfg.batch, n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


import ctypes as C
os.environ["PAFFT_FUSED"] = "0"
for i in range(plan.num_passes()):
    t = timeit(lambda: pf._check(pf.lib.pafft_convolve_permfree_pass(plan._h, filt._h, C.c_void_p(x.data_ptr()),
                                                                     C.c_void_p(y.data_ptr()), cfg.batch, i, None)))
    print(f"config {idx} pass {i} alone (3-launch kernel): {t:.3f} ms")
os.environ["PAFFT_FUSED"] = "1"
for i in range(3):
    os.environ["PAFFT_FUSED_ONLY"] = str(i)
    t = timeit(lambda: pf.convolve_permfree_out(x, y, filt, plan))
    print(f"config {idx} pass {i} alone (fused kernel):   {t:.3f} ms")
os.environ.pop("PAFFT_FUSED_ONLY")
print(f"config {idx} fused all: {timeit(lambda: pf.convolve_permfree_out(x, y, filt, plan)):.3f} ms")
