"""Seeded random plans on the GPU against the oracle: rank 1-3, a radix per
axis from {2, 3, 4, 5, 8}, extents r^t, batches 1-3, fp64 and fp32, random
forced pass schedules (PAFFT_MID_STAGES), through both the permutation-free
path and the standard-order comparator.  The bar is the north star's:
relative L2 <= 1e-12 (fp64) / 1e-5 (fp32) against the oracle on the same
inputs."""
import os

import numpy as np
import pytest

from helpers import rand_c, rel_l2

pytestmark = pytest.mark.gpu

RADICES = [2, 3, 4, 5, 8]
MAXLOG = {2: 12, 3: 8, 4: 6, 5: 6, 8: 4}


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    rank = int(rng.integers(1, 4))
    radices, dims = [], []
    budget = 15.0  # log2 of the total size
    for _ in range(rank):
        r = int(rng.choice(RADICES))
        tmax = max(0, min(MAXLOG[r], int(budget / np.log2(r))))
        t = int(rng.integers(0 if rank > 1 else 1, tmax + 1)) if tmax > 0 else 0
        radices.append(r)
        dims.append(r ** t)
        budget -= t * np.log2(r)
    batch = int(rng.integers(1, 4))
    f32 = bool(rng.random() < 0.3)
    mid = int(rng.integers(0, 4))  # 0 = default schedule
    return radices, dims, batch, f32, mid


CASES = [_case(s) for s in range(48)]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2506_12718_b200 as pf
    assert torch.cuda.is_available()
    return pf, torch


@pytest.mark.parametrize("radices,dims,batch,f32,mid", CASES, ids=[str(c) for c in CASES])
def test_random_plan_matches_oracle(env, orc, radices, dims, batch, f32, mid):
    pf, torch = env
    n = int(np.prod(dims))
    prec = pf.F32 if f32 else pf.F64
    cdt = torch.complex64 if f32 else torch.complex128
    bar = 1e-5 if f32 else 1e-12
    xs = np.stack([rand_c(n, 7 * n + b) for b in range(batch)])
    h = rand_c(n, 3 * n + 1)
    if f32:
        xs = xs.astype(np.complex64).astype(np.complex128)
        h = h.astype(np.complex64).astype(np.complex128)
    if mid:
        os.environ["PAFFT_MID_STAGES"] = str(mid)
    try:
        plan = pf.Plan(radices, dims, precision=prec)
    finally:
        os.environ.pop("PAFFT_MID_STAGES", None)
    op = orc.plan(list(radices), dims)
    g = op.filter_from_impulse(h)
    want = [op.convolve_permfree(xs[b], op.prepare_filter(g)) for b in range(batch)]
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    x = torch.from_numpy(xs).to("cuda", cdt)
    y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan).cpu().numpy().astype(np.complex128)
    assert max(rel_l2(y[b], want[b]) for b in range(batch)) <= bar
    # the standard-order comparator (two explicit reorderings) on the same inputs
    gd = torch.from_numpy(np.asarray(g).reshape(-1)).to("cuda", cdt)
    ys = pf.convolve_standard_(x.clone(), gd, plan).cpu().numpy().astype(np.complex128)
    assert max(rel_l2(ys[b], want[b]) for b in range(batch)) <= bar


def _case_large(seed):
    rng = np.random.default_rng(5000 + seed)
    rank = int(rng.integers(1, 4))
    radices, dims = [], []
    budget = 20.0
    for q in range(rank):
        r = int(rng.choice(RADICES))
        tmax = int(budget / np.log2(r))
        t = int(rng.integers(1 if q == 0 else 0, max(1, tmax) + 1)) if tmax > 0 else 0
        radices.append(r)
        dims.append(r ** t)
        budget -= t * np.log2(r)
    return radices, dims, int(rng.integers(1, 3)), bool(rng.random() < 0.3), bool(rng.random() < 0.5)


LARGE = [_case_large(s) for s in range(24)]


@pytest.mark.parametrize("radices,dims,batch,f32,inplace", LARGE, ids=[str(c) for c in LARGE])
def test_random_large_plan_matches_oracle(env, orc, radices, dims, batch, f32, inplace):
    """Up to 2^20 points per signal: multi-pass schedules on every axis, in place
    or out of place."""
    pf, torch = env
    n = int(np.prod(dims))
    prec = pf.F32 if f32 else pf.F64
    cdt = torch.complex64 if f32 else torch.complex128
    bar = 1e-5 if f32 else 1e-12
    xs = np.stack([rand_c(n, 11 * n + b) for b in range(batch)])
    h = rand_c(n, 5 * n + 3)
    if f32:
        xs = xs.astype(np.complex64).astype(np.complex128)
        h = h.astype(np.complex64).astype(np.complex128)
    plan = pf.Plan(radices, dims, precision=prec)
    op = orc.plan(list(radices), dims)
    gh = op.prepare_filter(op.filter_from_impulse(h))
    want = [op.convolve_permfree(xs[b], gh) for b in range(batch)]
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    x = torch.from_numpy(xs).to("cuda", cdt)
    if inplace:
        y = pf.convolve_permfree_(x, filt, plan)
    else:
        y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan)
    y = y.cpu().numpy().astype(np.complex128)
    assert max(rel_l2(y[b], want[b]) for b in range(batch)) <= bar


@pytest.mark.parametrize("radices,dims,batch,f32,mid", CASES[:32], ids=[str(c) for c in CASES[:32]])
def test_random_plan_transforms_match_oracle(env, orc, radices, dims, batch, f32, mid):
    """The device transforms of the same random plans (fp64): natural-order
    forward/backward, the bare ladders (A, A-bar, A^T) and the explicit
    permutation (bit-exact) against the oracle's (transform.cpp:8-26,
    butterfly.cpp:423-466, permutation.cpp:46-90)."""
    pf, torch = env
    n = int(np.prod(dims))
    xs = np.stack([rand_c(n, 13 * n + b) for b in range(batch)])
    plan = pf.Plan(radices, dims, precision=pf.F64)
    op = orc.plan(list(radices), dims)
    x = torch.from_numpy(xs).to("cuda", torch.complex128)

    def dev(fn):
        return fn(x.clone(), plan).cpu().numpy()

    def check(got, fn, bar=1e-12):
        for b in range(batch):
            assert rel_l2(got[b], fn(xs[b])) <= bar
    check(dev(pf.fft_forward_), op.fft_forward)
    check(dev(pf.fft_backward_), op.fft_backward)
    check(dev(pf.fft_transposed_), lambda v: op.butterfly_tensor(v, 2))
    check(dev(pf.fft_forward_unordered_), lambda v: op.butterfly_tensor(v, 0))
    check(dev(pf.fft_backward_unordered_), lambda v: op.butterfly_tensor(v, 1) / n)
    got = dev(pf.permute_)
    for b in range(batch):
        assert np.array_equal(got[b], op.permute(xs[b]))


@pytest.mark.parametrize("radices,dims,batch,f32,mid", CASES[:24], ids=[str(c) for c in CASES[:24]])
def test_random_plan_dropin_host_api(env, orc, radices, dims, batch, f32, mid):
    """The reference-shaped host API (numpy C-order arrays, module.cpp:73-149):
    prepare_filter is bit-exact (one permutation of the natural spectrum), the
    device-side prepare-from-impulse equals it, and convolve_permfree on host
    arrays matches the oracle."""
    pf, torch = env
    n = int(np.prod(dims))
    plan = pf.Plan(radices, dims, precision=pf.F64)
    op = orc.plan(list(radices), dims)
    h = rand_c(n, 17 * n + 1)
    g = op.filter_from_impulse(h)                       # vec order
    gh = op.prepare_filter(g)
    filt = pf.prepare_filter(g.reshape(dims, order="F"), plan)
    assert np.array_equal(filt.ghat, gh)
    fdev = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", torch.complex128), plan)
    assert rel_l2(fdev.ghat, gh) <= 1e-13
    x = rand_c(n, 19 * n + 2)
    y = pf.convolve_permfree(x.reshape(dims, order="F"), filt, plan)
    assert rel_l2(np.asarray(y).reshape(-1, order="F"), op.convolve_permfree(x, gh)) <= 1e-12


@pytest.mark.parametrize("radices,dims,batch,f32,mid", CASES[:24], ids=[str(c) for c in CASES[:24]])
def test_random_plan_host_buffer_path_bitwise(env, radices, dims, batch, f32, mid):
    """The host-buffer entry point (pinned H2D, convolve, D2H pipelined over
    streams; the e2e leg of bench.py) gives exactly the device path's result,
    fp32 odd lengths included."""
    pf, torch = env
    n = int(np.prod(dims))
    prec = pf.F32 if f32 else pf.F64
    cdt = torch.complex64 if f32 else torch.complex128
    xs = np.stack([rand_c(n, 23 * n + b) for b in range(batch)])
    h = rand_c(n, 29 * n + 1)
    plan = pf.Plan(radices, dims, precision=prec)
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    x = torch.from_numpy(xs).to(cdt)
    ydev = pf.convolve_permfree_out(x.cuda(), torch.empty_like(x, device="cuda"), filt, plan).cpu()
    xp = x.pin_memory()
    pf.convolve_permfree_host(xp.numpy(), filt, plan)  # in place on the pinned buffer
    assert torch.equal(xp, ydev)
