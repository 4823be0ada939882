"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the container that has /root/reference (oracle/_ref/libpafft_ref.so is
built from its sources by oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

For radix 2/4/8 the outputs come from pafft's own public API
(filter_from_impulse, prepare_filter, convolve_permfree, convolve_standard,
butterfly ladders, permute_tensor).  pafft cannot run radix 3/5
(core.hpp:14-19), so for those shapes the fixture holds pafft's radix-agnostic
direct O(N^2) sum (oracle::naive_circular_convolution, oracle.cpp:87-123) and
naive DFT (oracle.cpp:50-85) on the same inputs.  Inputs are seeded numpy
U(-1, 1) draws (seed recorded in each fixture).  Arrays are complex128 in vec
order (first index fastest).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

SHAPES_248 = [(2, [4]), (2, [64]), (2, [1024]), (2, [4096]), (4, [256]), (4, [1024]), (8, [512]),
              (2, [8, 4]), (2, [16, 16]), (2, [64, 64]), (4, [16, 16]), (4, [4, 64]), (8, [64, 8]),
              (2, [2, 2, 2, 2]), (2, [4, 2, 8]), (4, [4, 16, 4]), (4, [16, 4, 16]), (8, [8, 8, 8])]
SHAPES_35 = [(3, [3]), (3, [9]), (3, [243]), (3, [2187]), (5, [5]), (5, [125]), (5, [3125]), (3, [27, 81]),
             (3, [9, 9, 27]), (5, [25, 125]), (5, [5, 25])]


def rand(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def main():
    if not oracle.Ref.available():
        raise SystemExit("oracle/_ref/libpafft_ref.so missing: run `make -C oracle` where /root/reference exists")
    R = oracle.Ref()
    out = {}
    for radix, dims in SHAPES_248:
        n = int(np.prod(dims))
        seed = 1000 + n + 7 * radix + len(dims)
        x, h = rand(n, seed), rand(n, seed + 1)
        p = R.plan(radix, dims)
        g = p.filter_from_impulse(h)
        ghat = p.prepare_filter(g)
        key = f"r{radix}_" + "x".join(map(str, dims))
        out[key + "_x"] = x
        out[key + "_h"] = h
        out[key + "_g"] = g
        out[key + "_ghat"] = ghat
        out[key + "_permfree"] = p.convolve_permfree(x, ghat)
        out[key + "_standard"] = p.convolve_standard(x, g)
        out[key + "_transposed"] = p.butterfly_tensor(x, oracle.TRANSPOSED)
        out[key + "_forward"] = p.butterfly_tensor(x, oracle.FORWARD)
        out[key + "_conjugate"] = p.butterfly_tensor(x, oracle.CONJUGATE)
        out[key + "_permuted"] = p.permute(x)
        if n <= 1024:
            out[key + "_direct"] = R.naive_conv(x, h, dims)
        out[key + "_seed"] = np.array(seed)
    for radix, dims in SHAPES_35:
        n = int(np.prod(dims))
        seed = 2000 + n + 7 * radix + len(dims)
        x, h = rand(n, seed), rand(n, seed + 1)
        key = f"r{radix}_" + "x".join(map(str, dims))
        out[key + "_x"] = x
        out[key + "_h"] = h
        out[key + "_direct"] = R.naive_conv(x, h, dims)       # pafft oracle.cpp:87-123
        out[key + "_dft"] = R.naive_dft(h, dims)               # pafft oracle.cpp:50-85
        out[key + "_seed"] = np.array(seed)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB,", len(out), "arrays")


if __name__ == "__main__":
    main()
