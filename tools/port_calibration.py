"""CPU reference-arm calibration: pafft itself (oracle/_ref, radix 2) against
the two CPU stand-ins used where pafft cannot run (radix 3/5): the generic
oracle restatement and the reference-style specialised ladders
(oracle/fast_ladders.c).  Config 1 shape (2^20, radix 2), 1 and all threads."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2506_12718_b200 import workload  # noqa: E402


def main(nsig=8):
    cfg = workload.get_config(1)
    h = workload.impulse(cfg)
    xs = workload.signals(cfg, 0, nsig)
    threads = len(os.sched_getaffinity(0))
    R = oracle.Ref()
    rp = R.plan(cfg.radix, cfg.dims)
    b = rp.batch(rp.prepare_filter(rp.filter_from_impulse(h)), xs)
    O = oracle.Oracle()
    op = O.plan(cfg.radix, cfg.dims)
    gh = op.prepare_filter(op.filter_from_impulse(h))
    gr, gi = np.ascontiguousarray(gh.real), np.ascontiguousarray(gh.imag)
    for th in (1, threads):
        print(f"threads={th}: pafft {nsig / b.run(th):.2f} conv/s", end="")
        for name, fn in (("oracle", op.convolve_permfree_batch_split), ("fast", op.convolve_permfree_fast_batch_split)):
            re, im = np.ascontiguousarray(xs.real), np.ascontiguousarray(xs.imag)
            t = time.perf_counter()
            fn(gr, gi, re, im, nsig, th)
            print(f", {name} {nsig / (time.perf_counter() - t):.2f} conv/s", end="")
        print()


if __name__ == "__main__":
    main()
