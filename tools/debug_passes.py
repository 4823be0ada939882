"""Per-ladder GPU-vs-oracle errors for multi-pass plans (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2506_12718_b200 as pf

O = oracle.Oracle()
cases = [(2, [1 << 16]), (2, [1 << 13]), (3, [3 ** 8]), (4, [4 ** 7]), (5, [5 ** 6]), (2, [64, 128]), (3, [3**13])]
for mid, st in [(None, None), ("3", "2")]:
    if mid:
        os.environ["PAFFT_MAX_MID_STAGES"] = mid; os.environ["PAFFT_MAX_STRIDED_STAGES"] = st
    for radix, dims in cases:
        n = int(np.prod(dims))
        rng = np.random.default_rng(0)
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        op = O.plan(radix, dims)
        plan = pf.Plan(radix, dims)
        xa = x.reshape(dims, order="F")
        res = {}
        for name, fn, var in [("DIF(A^T)", pf.fft_transposed, oracle.TRANSPOSED), ("DIT(A)", pf.fft_forward_unordered, oracle.FORWARD)]:
            y = fn(xa, plan).ravel(order="F")
            ref = op.butterfly_tensor(x, var)
            res[name] = oracle.rel_l2(y, ref)
        yb = pf.fft_backward_unordered(xa, plan).ravel(order="F")
        res["DIT(Abar)/N"] = oracle.rel_l2(yb, op.butterfly_tensor(x, oracle.CONJUGATE) / n)
        g = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        ghat = op.prepare_filter(g)
        f = pf.prepare_filter(g.reshape(dims, order="F"), plan)
        res["permfree"] = oracle.rel_l2(pf.convolve_permfree(xa, f, plan).ravel(order="F"), op.convolve_permfree(x, ghat))
        print(radix, dims, mid, {k: f"{v:.2e}" for k, v in res.items()})
        print("   ", plan.describe().replace("\n", "\n    "))
