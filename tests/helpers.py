"""Shared test helpers: seeded inputs and error metrics."""
import numpy as np


def rand_c(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def rel_l2(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def max_diff(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return float(max(np.abs(a.real - b.real).max(initial=0), np.abs(a.imag - b.imag).max(initial=0)))


def transform_tolerance(n, max_abs_x):
    """tolerance.hpp:12-14"""
    return 1e-12 * np.log2(n) * max_abs_x


def convolution_tolerance(n, max_abs_x, max_abs_h):
    """tolerance.hpp:18-20"""
    return 1e-10 * np.sqrt(n) * max_abs_x * max_abs_h


# Shapes: the reference's verification grid (verify.cpp:13-44) plus radix 3/5.
GRID = (
    [(2, [n]) for n in [2 ** k for k in range(1, 13)]]
    + [(4, [n]) for n in [4 ** k for k in range(1, 7)]]
    + [(8, [n]) for n in [8, 64, 512, 4096]]
    + [(2, d) for d in ([2, 2], [4, 8], [8, 4], [32, 2], [16, 16], [2, 64], [64, 64])]
    + [(4, d) for d in ([4, 4], [16, 4], [4, 16], [16, 16], [4, 64], [64, 64])]
    + [(8, d) for d in ([8, 8], [64, 8], [8, 64], [64, 64])]
    + [(2, d) for d in ([2, 2, 2], [4, 2, 8], [8, 8, 8], [2, 16, 4], [16, 16, 16])]
    + [(4, d) for d in ([4, 4, 4], [16, 4, 4], [4, 16, 16], [16, 16, 16])]
    + [(8, [8, 8, 8])]
)
GRID_ODD = (
    [(3, [3 ** k]) for k in range(1, 9)]
    + [(5, [5 ** k]) for k in range(1, 6)]
    + [(3, d) for d in ([27, 81], [9, 9, 27], [3, 243], [81, 3])]
    + [(5, d) for d in ([25, 125], [5, 25], [125, 5, 5])]
)

# Per-axis radices: axis q is a power of radices[q].
GRID_MIXED = [
    ([3, 2], [27, 64]), ([2, 3], [64, 81]), ([5, 4], [25, 64]), ([4, 5], [256, 25]), ([2, 3, 5], [8, 9, 25]),
    ([8, 3], [64, 27]), ([4, 5, 3], [16, 5, 9]), ([3, 8], [243, 8]), ([5, 2], [125, 32]), ([2, 4], [32, 16]),
]
