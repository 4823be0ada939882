"""Relative L2 error vs the oracle on one or two signals of each BASELINE
config (fp64), to see the margin below the north star's 1e-12.
usage: [PAFFT_LIB=ab/libX.so] python tools/accuracy_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2506_12718_b200 as pf
from paper_2506_12718_b200 import workload

orc = oracle.Oracle()
for idx in (1, 2, 3, 4, 5):
    cfg = workload.get_config(idx, "f64")
    plan = pf.Plan(cfg.radix, cfg.dims, precision=pf.F64)
    h = workload.impulse(cfg)
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", torch.complex128), plan)
    nb = 2 if idx != 4 else 1
    xs = workload.signals(cfg, 0, nb)
    x = torch.from_numpy(xs).to("cuda", torch.complex128).reshape(nb, -1)
    y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan).cpu().numpy()
    op = orc.plan(cfg.radix, cfg.dims)
    gh = op.prepare_filter(op.filter_from_impulse(h))
    errs = [oracle.rel_l2(y[b], op.convolve_permfree(xs[b].reshape(-1), gh)) for b in range(nb)]
    print(f"config {idx}: rel_l2 vs oracle " + " ".join(f"{e:.2e}" for e in errs), flush=True)
