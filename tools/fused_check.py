"""Fused single-launch convolution vs the three-launch path: bitwise equality
of the results and device time per step (CUDA events).
usage: python tools/fused_check.py [config ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2506_12718_b200 as pf
from paper_2506_12718_b200 import workload


def run(cfg_idx, batch=0, reps=10):
    cfg = workload.get_config(cfg_idx, "f64")
    plan = pf.Plan(cfg.radix, cfg.dims, precision=pf.F64)
    h = workload.impulse(cfg)
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", torch.complex128), plan)
    b = batch or cfg.batch
    n = int(torch.tensor(cfg.dims).prod())
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(b, n, dtype=torch.complex128, device="cuda", generator=g)
    out = {}
    for mode in ("0", "1"):
        os.environ["PAFFT_FUSED"] = mode
        y = torch.empty_like(x)
        pf.convolve_permfree_out(x, y, filt, plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            pf.convolve_permfree_out(x, y, filt, plan)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = (y.clone(), e0.elapsed_time(e1) / reps)
    y0, t0 = out["0"]
    y1, t1 = out["1"]
    same = torch.equal(y0, y1)
    err = ((y0 - y1).abs().pow(2).sum() / y0.abs().pow(2).sum()).sqrt().item()
    print(f"config {cfg_idx} batch {b}: bitwise_equal={same} rel_l2={err:.2e} "
          f"3-launch {t0:.3f} ms  fused {t1:.3f} ms  speedup {t0 / t1:.3f}", flush=True)


if __name__ == "__main__":
    # args: config[:batch][@lag] ...
    for c in (sys.argv[1:] or ["2", "5", "1"]):
        c, _, lag = c.partition("@")
        if lag:
            os.environ["PAFFT_FUSED_LAG"] = lag
        else:
            os.environ.pop("PAFFT_FUSED_LAG", None)
        idx, _, b = c.partition(":")
        print(f"lag={lag or 'auto'} ", end="")
        run(int(idx), int(b or 0))
