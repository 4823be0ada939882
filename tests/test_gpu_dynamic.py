"""Dynamic tile order of the persistent pass kernels (pass.cuh, PassArgs::ctr):
launches with several tiles per CTA hand tiles out through a per-stream
counter instead of the static round-robin order.  Every tile is independent
(convolution.cpp:45-52 applies the same ladders to every signal), so the result
must be bitwise the static one; launches inside a CUDA-graph capture and on the
per-thread default stream keep the static order; concurrent streams each have
their own counter pair, which every launch leaves zeroed."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2506_12718_b200 as pf
    return pf


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _data(torch, pf, n, batch, prec, seed):
    rng = np.random.default_rng(seed)
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    x = torch.from_numpy(rng.uniform(-1, 1, (batch, n)) + 1j * rng.uniform(-1, 1, (batch, n))).to("cuda", cdt)
    h = torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n)).to("cuda", cdt)
    return x, h


CASES = [
    # radix, dims, batch, precision, forced CONV stages (0 = default), max strided stages
    (3, [2187], 1500, "f64", 0, 0),      # one contiguous CONV pass, 1500 tiles
    (3, [6561], 400, "f64", 4, 2),       # strided DIF/DIT with external twiddles + CONV
    (5, [3125], 600, "f32", 3, 2),       # fp32 strided tiles (per-row shifted layout, register stores)
    (2, [4096], 900, "f64", 6, 3),       # swizzled power-of-two CONV tiles, two strided passes each way
    (2, [64, 128, 8], 24, "f64", 0, 0),  # per-axis passes of a 3-D plan
    (4, [256, 64], 40, "f32", 0, 0),
]


@pytest.mark.parametrize("radix,dims,batch,prec,mid,strided", CASES)
def test_dynamic_tile_order_is_bitwise_the_static_one(pf, torch, monkeypatch, radix, dims, batch, prec, mid, strided):
    if mid:
        monkeypatch.setenv("PAFFT_MID_STAGES", str(mid))
    if strided:
        monkeypatch.setenv("PAFFT_MAX_STRIDED_STAGES", str(strided))
    precision = pf.F64 if prec == "f64" else pf.F32
    plan = pf.Plan(radix, dims, precision=precision)
    x, h = _data(torch, pf, plan.total, batch, precision, 5)
    filt = pf.prepare_filter_from_impulse(h, plan)
    monkeypatch.setenv("PAFFT_DYN_MIN_TILES", "0")
    d0 = pf.dynamic_launch_count()
    y_static = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan)
    torch.cuda.synchronize()
    assert pf.dynamic_launch_count() == d0
    monkeypatch.setenv("PAFFT_DYN_MIN_TILES", "1")
    monkeypatch.setenv("PAFFT_DYN_MIN_OCC", "1")
    for _ in range(3):  # repeated launches reuse the stream's counter pair: each must leave it zeroed
        y_dyn = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan)
        torch.cuda.synchronize()
        assert torch.equal(y_dyn, y_static), plan.describe()
    assert pf.dynamic_launch_count() == d0 + 3 * max(plan.num_passes(), 0)
    # in place as well
    xin = x.clone()
    pf.convolve_permfree_(xin, filt, plan)
    torch.cuda.synchronize()
    assert torch.equal(xin, y_static)


def test_graph_capture_keeps_the_static_order(pf, torch, monkeypatch):
    plan = pf.Plan(3, [2187])
    x, h = _data(torch, pf, plan.total, 1200, pf.F64, 7)
    filt = pf.prepare_filter_from_impulse(h, plan)
    monkeypatch.setenv("PAFFT_DYN_MIN_TILES", "1")
    monkeypatch.setenv("PAFFT_DYN_MIN_OCC", "1")
    want = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan)
    torch.cuda.synchronize()
    y = torch.empty_like(x)
    d0 = pf.dynamic_launch_count()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            pf.convolve_permfree_out(x, y, filt, plan, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    assert pf.dynamic_launch_count() == d0  # a captured launch may replay on any stream: static order
    for _ in range(2):
        y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, want)


def test_concurrent_streams_have_their_own_counters(pf, torch, monkeypatch):
    monkeypatch.setenv("PAFFT_MID_STAGES", "4")
    monkeypatch.setenv("PAFFT_MAX_STRIDED_STAGES", "2")
    plan = pf.Plan(3, [6561])
    nthreads, rounds = 4, 8
    data = [_data(torch, pf, plan.total, 300, pf.F64, 20 + t) for t in range(nthreads)]
    filt = pf.prepare_filter_from_impulse(data[0][1], plan)
    monkeypatch.setenv("PAFFT_DYN_MIN_TILES", "0")
    want = [pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan) for x, _ in data]
    torch.cuda.synchronize()
    monkeypatch.setenv("PAFFT_DYN_MIN_TILES", "1")
    monkeypatch.setenv("PAFFT_DYN_MIN_OCC", "1")
    errors, ok = [], [0] * nthreads

    def runner(t):
        try:
            s = torch.cuda.Stream()
            x = data[t][0]
            with torch.cuda.stream(s):
                for _ in range(rounds):
                    y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan, stream=s)
                    s.synchronize()
                    ok[t] += int(torch.equal(y, want[t]))
        except Exception as e:  # surfaced below
            errors.append(e)

    ths = [threading.Thread(target=runner, args=(t,)) for t in range(nthreads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
    assert ok == [rounds] * nthreads
