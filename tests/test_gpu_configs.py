"""BASELINE.json configurations at full size on the GPU.

Each config is checked three ways: (1) EVERY signal of the full BASELINE
batch (config 1: all 100 batch-1 calls; 64 / 16 / 8 / 4096 for configs 2-5),
in fp64 and fp32, against the CPU reference on the same seeded signals --
for radix 2/4 (configs 1, 3, 4) that is pafft itself (oracle/_ref, the
reference library compiled from its own sources), for radix 3/5 (configs 2, 5,
not representable in pafft) the pinned restatement (oracle/pafft_oracle.c),
run threaded over the batch; relative L2 <= 1e-12 fp64 / 1e-5 fp32 per
signal and over the batch (north_star; fp32 against the fp64 pipeline on the
fp32-rounded inputs); (2) size-independent properties over the
whole batch -- a delta filter reproduces the input, a shifted delta shifts it
cyclically, the map is linear, repeated calls are bitwise identical; (3) the
C++ drop-in program (tests/cpp/test_dropin.cpp) runs the reference's own unit
cases against the GPU library.
"""
import os
import subprocess

import numpy as np
import pytest

from helpers import rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pf():
    import paper_2506_12718_b200 as pf
    return pf


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _setup(pf, torch, cfg, batch):
    from paper_2506_12718_b200 import workload
    prec = pf.F64 if cfg.precision == "f64" else pf.F32
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    plan = pf.Plan(cfg.radix, cfg.dims, precision=prec)
    h = workload.impulse(cfg)
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    xs = workload.signals(cfg, 0, batch) if batch else None
    return plan, filt, h, xs, cdt


def _cpu_reference(orc, cfg, hin, threads):
    """Returns (kind, run(xin) -> y) for the config: pafft itself (oracle/_ref)
    for radix 2/4/8, the pinned restatement for radix 3/5."""
    import oracle
    if cfg.radix in (2, 4, 8) and oracle.Ref.available():
        rp = oracle.Ref().plan(cfg.radix, cfg.dims)
        ghat = rp.prepare_filter(rp.filter_from_impulse(hin))

        def run(xin):
            b = rp.batch_split(ghat, np.ascontiguousarray(xin.real), np.ascontiguousarray(xin.imag))
            b.run(threads)
            return np.stack([b.read(i) for i in range(len(xin))])
        return "pafft (oracle/_ref)", run
    op = orc.plan(cfg.radix, cfg.dims)
    ghat = op.prepare_filter(op.filter_from_impulse(hin))
    gr, gi = np.ascontiguousarray(ghat.real), np.ascontiguousarray(ghat.imag)

    def run(xin):
        re, im = np.ascontiguousarray(xin.real), np.ascontiguousarray(xin.imag)
        op.convolve_permfree_batch_split(gr, gi, re, im, len(xin), threads)
        return re + 1j * im
    return "restatement (oracle/pafft_oracle.c)", run


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_config_full_batch_matches_reference(pf, torch, orc, idx, prec):
    """Every signal of the BASELINE batch against the CPU reference."""
    from paper_2506_12718_b200 import workload
    cfg = workload.get_config(idx, prec)
    count = cfg.calls if cfg.calls > 1 else cfg.batch
    plan, filt, h, _, cdt = _setup(pf, torch, cfg, 0)
    hin = h.astype(np.complex64).astype(np.complex128) if prec == "f32" else h
    threads = len(os.sched_getaffinity(0))
    kind, cpu_conv = _cpu_reference(orc, cfg, hin, threads)
    bar = 1e-12 if prec == "f64" else 1e-5
    chunk = max(1, min(count, (1 << 30) // (16 * cfg.total)))  # <= 1 GiB of fp64 signals at a time
    num = den = 0.0
    worst = 0.0
    for c0 in range(0, count, chunk):
        n = min(chunk, count - c0)
        xs = workload.signals(cfg, c0, n)
        xin = xs.astype(np.complex64).astype(np.complex128) if prec == "f32" else xs
        x = torch.from_numpy(xs).to("cuda", cdt)
        y = torch.empty_like(x)
        if cfg.calls > 1:  # config 1: each signal is its own batch-1 call
            for b in range(n):
                pf.convolve_permfree_out(x[b:b + 1], y[b:b + 1], filt, plan)
        else:
            pf.convolve_permfree_out(x, y, filt, plan)
        torch.cuda.synchronize()
        yg = y.cpu().numpy().astype(np.complex128)
        del x, y
        want = cpu_conv(xin)
        for b in range(n):
            e = rel_l2(yg[b], want[b])
            worst = max(worst, e)
            assert e <= bar, (idx, prec, c0 + b, e, kind)
        num += float(np.sum(np.abs(yg - want) ** 2))
        den += float(np.sum(np.abs(want) ** 2))
    whole = (num / den) ** 0.5
    print(f"config {idx} {prec}: {count} signals vs {kind}: batch rel_l2 {whole:.3e}, worst signal {worst:.3e}")
    assert whole <= bar


@pytest.mark.parametrize("idx", [2, 3, 4, 5])
def test_config_properties_full_batch(pf, torch, idx):
    """delta -> identity, shifted delta -> cyclic shift, linearity, determinism."""
    from paper_2506_12718_b200 import workload
    cfg = workload.get_config(idx)
    batch = cfg.batch  # the whole BASELINE batch
    plan = pf.Plan(cfg.radix, cfg.dims)
    n = cfg.total
    xs = torch.from_numpy(workload.signals(cfg, 0, batch)).cuda()
    # identity
    d = np.zeros(n, complex)
    d[0] = 1
    f_id = pf.prepare_filter_from_impulse(torch.from_numpy(d).cuda(), plan)
    y = pf.convolve_permfree_out(xs, torch.empty_like(xs), f_id, plan)
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy(), xs.cpu().numpy()) <= 1e-13
    # cyclic shift by s along axis 0 (and 1 for 2-D)
    s = 5
    d2 = np.zeros(n, complex)
    d2[s] = 1
    f_sh = pf.prepare_filter_from_impulse(torch.from_numpy(d2).cuda(), plan)
    y2 = pf.convolve_permfree_out(xs, torch.empty_like(xs), f_sh, plan).cpu().numpy()
    xv = xs.cpu().numpy()
    dims = cfg.dims
    want = np.roll(xv.reshape([batch] + dims[::-1]), s, axis=len(dims)).reshape(batch, n)
    assert rel_l2(y2, want) <= 1e-13
    # linearity with the config's own filter
    f = pf.prepare_filter_from_impulse(torch.from_numpy(workload.impulse(cfg)).cuda(), plan)
    a, b = 0.7 - 1.3j, -0.2 + 0.5j
    x1, x2 = xs[: batch // 2], xs[batch // 2: 2 * (batch // 2)]
    lhs = pf.convolve_permfree_out(a * x1 + b * x2, torch.empty_like(x1), f, plan)
    r1 = pf.convolve_permfree_out(x1, torch.empty_like(x1), f, plan)
    r2 = pf.convolve_permfree_out(x2, torch.empty_like(x2), f, plan)
    assert rel_l2(lhs.cpu().numpy(), (a * r1 + b * r2).cpu().numpy()) <= 1e-13
    # determinism (reuse without drift, test_convolution.cpp:99-111)
    again = pf.convolve_permfree_out(x1, torch.empty_like(x1), f, plan)
    torch.cuda.synchronize()
    assert torch.equal(again, r1)


def test_standard_path_matches_permfree_at_config2(pf, torch):
    """The standard-order GPU comparator (two permutations) agrees with the
    permutation-free path (north_star item 5) and costs exactly 2 passes."""
    from paper_2506_12718_b200 import workload
    cfg = workload.get_config(2)
    plan = pf.Plan(cfg.radix, cfg.dims)
    h = torch.from_numpy(workload.impulse(cfg)).cuda()
    f = pf.prepare_filter_from_impulse(h, plan)
    g = h.clone()
    pf.fft_forward_(g, plan)  # natural-order spectrum
    x = torch.from_numpy(workload.signals(cfg, 0, 2)).cuda()
    ys = x.clone()
    pf.reset_permutation_pass_count()
    pf.convolve_standard_(ys, g, plan)
    torch.cuda.synchronize()
    assert pf.permutation_pass_count() == 2 * 2  # two per signal
    yp = pf.convolve_permfree_out(x, torch.empty_like(x), f, plan)
    torch.cuda.synchronize()
    assert rel_l2(ys.cpu().numpy(), yp.cpu().numpy()) <= 1e-13


def test_cpp_dropin_program():
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    src = exe + ".cpp"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L" + os.path.join(ROOT, "paper_2506_12718_b200"), "-lpafft_b200",
                        "-Wl,-rpath," + os.path.join(ROOT, "paper_2506_12718_b200"),
                        "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
