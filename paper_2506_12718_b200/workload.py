"""BASELINE.json workloads (synthetic, seeded) and their roofline figures.

Inputs follow SURVEY.md 8(d): SplitMix64 (bench.cpp:22-42), U(-1,1) as in
bench.cpp:36-49, N(0,1) by Box-Muller; re then im per element; filter seed =
base + 1 (bench.cpp:145 convention), signal b seed = base + 2 + b; base =
0x5eed5eed5eed5eed (bench.hpp:32).  The "filter" is the impulse response h;
the device prepares ghat = A^T h (= P DFT(h)) outside any timed region.
All arrays are complex128 in vec order (first index fastest).
"""
from __future__ import annotations

import concurrent.futures as cf
import math
import os
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 0x5EED5EED5EED5EED
MASK64 = (1 << 64) - 1


@dataclass
class Config:
    idx: int
    name: str
    radix: int
    dims: list
    batch: int
    signal: str            # "uniform" | "normal"
    filt: str              # "cnormal" | "gauss2d" | "exp3d"
    calls: int = 1         # config 1: sequential batch-1 calls per step
    precision: str = "f64"
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def total(self):
        return int(np.prod(self.dims))

    @property
    def stages(self):
        return [round(math.log(d, self.radix)) for d in self.dims]


CONFIGS = {
    1: Config(1, "1d_2^20_r2_x100", 2, [1 << 20], 1, "uniform", "cnormal", calls=100,
              note="n=2^20 complex fp64, radix 2, fixed filter applied to 100 fresh signals, batch 1"),
    2: Config(2, "1d_3^13_r3_b64", 3, [3 ** 13], 64, "uniform", "cnormal",
              note="n=3^13 complex fp64, radix 3, batch 64"),
    3: Config(3, "2d_2048^2_r2_b16", 2, [2048, 2048], 16, "uniform", "gauss2d",
              note="2048x2048 complex fp64, radix 2 both axes, batch 16, Gaussian sigma=8"),
    4: Config(4, "3d_256^3_r4_b8", 4, [256, 256, 256], 8, "normal", "exp3d",
              note="256^3 complex fp64, radix 4, batch 8, exp(-|d|/16) kernel"),
    5: Config(5, "1d_5^7_r5_b4096", 5, [5 ** 7], 4096, "uniform", "cnormal",
              note="n=5^7 complex, radix 5, batch 4096"),
}


def get_config(idx: int, precision: str = "f64") -> Config:
    c = CONFIGS[int(idx)]
    if precision != c.precision:
        c = Config(**{**c.__dict__, "precision": precision, "extra": dict(c.extra)})
    return c


def seed_filter():
    return (BASE_SEED + 1) & MASK64


def seed_signal(b):
    return (BASE_SEED + 2 + b) & MASK64


def _pf():
    import paper_2506_12718_b200 as pf
    return pf


def impulse(cfg: Config, fill_normal=None) -> np.ndarray:
    """The filter's impulse response h (vec order, complex128).  `fill_normal`
    (seed, n) -> complex128 defaults to the product library's SplitMix64
    generator; the reference arm of bench.py passes the oracle's, which emits
    the same bytes (tests/test_abi.py), so that process never maps this package's
    library."""
    n = cfg.total
    if cfg.filt == "cnormal":
        return (fill_normal or _pf().fill_normal)(seed_filter(), n)
    if cfg.filt == "gauss2d":
        n1, n2 = cfg.dims
        d1 = np.minimum(np.arange(n1), n1 - np.arange(n1)).astype(np.float64)
        d2 = np.minimum(np.arange(n2), n2 - np.arange(n2)).astype(np.float64)
        sigma = 8.0
        h = np.exp(-(d1[:, None] ** 2 + d2[None, :] ** 2) / (2 * sigma * sigma))  # [i1, i2]
        h /= h.sum()
        return h.ravel(order="F").astype(np.complex128)  # vec: i1 fastest
    if cfg.filt == "exp3d":
        ds = [np.minimum(np.arange(n), n - np.arange(n)).astype(np.float64) for n in cfg.dims]
        r = np.sqrt(ds[0][:, None, None] ** 2 + ds[1][None, :, None] ** 2 + ds[2][None, None, :] ** 2)
        return np.exp(-r / 16.0).ravel(order="F").astype(np.complex128)
    raise ValueError(cfg.filt)


def signals(cfg: Config, first: int, count: int, out: np.ndarray | None = None, threads: int | None = None):
    """Signals first..first+count-1 as a (count, N) complex128 array (or into `out`,
    which may be a pinned numpy view).  Generated in parallel across signals."""
    pf = _pf()
    n = cfg.total
    if out is None:
        out = np.empty((count, n), dtype=np.complex128)
    fill = pf.fill_uniform if cfg.signal == "uniform" else pf.fill_normal
    lib = pf.lib
    import ctypes as C
    dp = C.POINTER(C.c_double)
    fn = lib.pafft_fill_uniform if cfg.signal == "uniform" else lib.pafft_fill_normal

    def one(i):
        row = out[i]
        fn(seed_signal(first + i), n, row.ctypes.data_as(dp))

    threads = threads or min(count, os.cpu_count() or 4)
    if count == 1:
        one(0)
    else:
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(count)))
    del fill
    return out


# ---------------------------------------------------------------- rooflines
CORE_FLOPS = {2: 4, 3: 16, 4: 16, 5: 48, 8: 0}


def flops_per_conv(cfg: Config) -> float:
    """F_alg = 2 F_FFT + 6N; F_FFT = N sum_q t_q (core_r + 6(r-1))/r.
    Radix 2/4 equal pafft's estimate_flop (bench.cpp:111-117)."""
    r = cfg.radix
    per = {2: 5.0, 4: 8.5, 3: (16 + 12) / 3, 5: (48 + 24) / 5, 8: 4.08 * 3}[r]
    t = sum(cfg.stages)
    return 2.0 * cfg.total * t * per + 6.0 * cfg.total


def signal_bytes(cfg: Config) -> int:
    return cfg.total * (16 if cfg.precision == "f64" else 8)


def shard_count(cfg: Config, gpus: int = 1, weak: bool = False) -> int:
    """B_g: convolutions per GPU sharing one resident ghat.
    Batched configs split the fixed global batch (batch / G, the largest shard
    when G does not divide it); config 1's call sequence runs as replicas."""
    if cfg.calls > 1:
        return cfg.calls
    if weak:
        return max(1, cfg.batch)
    return max(1, -(-cfg.batch // max(1, gpus)))


def bytes_per_conv(cfg: Config, gpus: int = 1, weak: bool = False) -> float:
    """B_alg = 2 S + S / B_g: read x once, write y once, ghat once per GPU per step."""
    S = signal_bytes(cfg)
    return 2.0 * S + S / shard_count(cfg, gpus, weak)
