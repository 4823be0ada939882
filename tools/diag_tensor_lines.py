"""Which (shape, variant) of the reference's 'tensor driver applies the 1-D
ladders along every mode' (test_butterfly.cpp:198-215) differ bitwise, and on
which axis: butterfly_tensor vs the 1-D ladder run line by line."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2506_12718_b200 as pf
import ctypes as C

OPS = {"forward": 2, "transposed": 4, "conjugate": 6}


def run(op, x, plan):
    re, im = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    pf._check(pf.lib.pafft_transform_split(plan._h, op, re.ctypes.data_as(C.POINTER(C.c_double)),
                                           im.ctypes.data_as(C.POINTER(C.c_double)), 1))
    return re + 1j * im


for radix, dims in [(2, [4, 8]), (4, [16, 4, 16]), (8, [8, 64]), (2, [2, 2, 2, 2])]:
    plan = pf.Plan(radix, dims)
    n = int(np.prod(dims))
    rng = np.random.default_rng(47)
    x0 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    print(radix, dims, plan.describe().replace("\n", " | "))
    for name, op in OPS.items():
        a = run(op, x0, plan)
        b = x0.reshape(dims[::-1]).copy()  # C-order view [i_{d-1}]...[i_0] of the vec buffer
        for q in range(len(dims)):
            lp = pf.Plan(radix, [dims[q]])
            ax = len(dims) - 1 - q
            moved = np.moveaxis(b, ax, -1)
            flat = moved.reshape(-1, dims[q])
            for i in range(flat.shape[0]):
                flat[i] = run(op, flat[i].copy(), lp)
            b = np.moveaxis(flat.reshape(moved.shape), -1, ax)
            # after axis q: compare with a tensor plan restricted... report running diff
        d = np.abs(a - b.reshape(-1)).max()
        print(f"   {name:10s} max|tensor - lines| = {d:.3e}")
