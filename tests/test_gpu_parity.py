"""GPU parity: the sm_100a path against the oracle (CPU restatement, pinned to
the reference in tests/test_oracle_pins.py) on the same seeded inputs.

Bars (north_star): relative L2 <= 1e-12 in fp64, <= 1e-5 in fp32; plus the
reference's own absolute tolerances (tolerance.hpp) against the direct sum.
Mirrors test_convolution.cpp:22-145 and verify.cpp:106-141.
"""
import os

import numpy as np
import pytest

from helpers import GRID, GRID_ODD, convolution_tolerance, max_diff, rand_c, rel_l2, transform_tolerance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2506_12718_b200 as pf
    return pf


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def dev_conv(pf, torch, plan, filt, x_vec, batch=1):
    t = torch.from_numpy(np.ascontiguousarray(x_vec)).cuda()
    pf.convolve_permfree_(t, filt, plan)
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _oracle_conv(orc, radix, dims, x, h):
    op = orc.plan(radix, dims)
    g = op.filter_from_impulse(h)
    return op.convolve_permfree(x, op.prepare_filter(g)), g, op


@pytest.mark.parametrize("radix,dims", GRID + GRID_ODD, ids=lambda v: str(v))
def test_permfree_matches_oracle_and_direct_sum(pf, torch, orc, radix, dims):
    n = int(np.prod(dims))
    x = rand_c(n, 89 + n)
    h = rand_c(n, 90 + n)
    y_orc, g, _ = _oracle_conv(orc, radix, dims, x, h)
    plan = pf.Plan(radix, dims)
    # device spectrum g (natural order, vec) -> prepared filter (one device permutation)
    gt = torch.from_numpy(g).cuda()
    filt = pf.prepare_filter_device(gt, plan)
    y = dev_conv(pf, torch, plan, filt, x)
    assert rel_l2(y, y_orc) <= 1e-12
    if n <= 4096:
        direct = orc.naive_conv(x, h, dims)
        tol = convolution_tolerance(n, np.abs(x).max(), np.abs(h).max())
        assert max_diff(y, direct) <= tol


@pytest.mark.parametrize("radix,dims", [(2, [64]), (3, [243]), (5, [125]), (2, [16, 32]), (3, [9, 27]),
                                        (4, [16, 16, 16]), (5, [25, 125]), (8, [512]), (3, [2187])])
def test_permfree_fp32(pf, torch, orc, radix, dims):
    n = int(np.prod(dims))
    x = rand_c(n, 7 + n).astype(np.complex64)
    h = rand_c(n, 8 + n).astype(np.complex64)
    # oracle: fp64 pipeline on the fp32-rounded inputs
    y_orc, g, _ = _oracle_conv(orc, radix, dims, x.astype(np.complex128), h.astype(np.complex128))
    plan = pf.Plan(radix, dims, precision=pf.F32)
    filt = pf.prepare_filter_device(torch.from_numpy(g.astype(np.complex64)).cuda(), plan)
    y = dev_conv(pf, torch, plan, filt, x)
    assert rel_l2(y, y_orc) <= 1e-5


def test_host_split_api_matches_reference_pipeline(pf, orc):
    """module.cpp-style numpy API: C-order arrays, pafft dims == numpy axes."""
    rng = np.random.default_rng(4)
    shape = (16, 16)
    x = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
    h = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
    expected = np.fft.ifftn(np.fft.fftn(x) * np.fft.fftn(h))
    plan = pf.Plan(2, list(shape))
    g = pf.filter_from_impulse(h, plan)
    np.testing.assert_allclose(g, np.fft.fftn(h), rtol=0, atol=1e-10)
    np.testing.assert_allclose(pf.convolve_standard(x, g, plan), expected, rtol=0, atol=1e-10)
    prepared = pf.prepare_filter(g, plan)
    np.testing.assert_allclose(pf.convolve_permfree(x, prepared, plan), expected, rtol=0, atol=1e-10)


def test_delay_filter_known_answer(pf):
    """test_convolution.cpp:41-61: the one-sample delay."""
    plan = pf.Plan(2, [4])
    g = pf.filter_from_impulse(np.array([0, 1, 0, 0], dtype=complex), plan)
    assert max_diff(g, np.array([1, -1j, -1, 1j])) < 1e-14
    x = np.array([1, 2, 3, 4], dtype=complex)
    assert max_diff(pf.convolve_standard(x, g, plan), [4, 1, 2, 3]) < 1e-13
    assert max_diff(pf.convolve_permfree(x, pf.prepare_filter(g, plan), plan), [4, 1, 2, 3]) < 1e-13


def test_prepare_filter_layout_bit_exact(pf):
    """test_convolution.cpp:32-39: prepare_filter([0,1,2,3]) == [0,2,1,3] exactly."""
    plan = pf.Plan(2, [4])
    f = pf.prepare_filter(np.array([0, 1, 2, 3], dtype=complex), plan)
    assert np.array_equal(f.ghat, np.array([0, 2, 1, 3], dtype=complex))
    assert f.key == plan.key()
    with pytest.raises(RuntimeError):
        pf.prepare_filter(np.zeros(3, dtype=complex), plan)


def test_pass_accounting(pf):
    """test_convolution.cpp:63-79: standard = 2, prepare = 1, permfree = 0."""
    plan = pf.Plan(4, [16, 16])
    g = rand_c(256, 73).reshape(16, 16, order="F")
    x = rand_c(256, 74).reshape(16, 16, order="F")
    pf.reset_permutation_pass_count()
    pf.convolve_standard(x, g, plan)
    assert pf.permutation_pass_count() == 2
    pf.reset_permutation_pass_count()
    filt = pf.prepare_filter(g, plan)
    assert pf.permutation_pass_count() == 1
    pf.reset_permutation_pass_count()
    pf.convolve_permfree(x, filt, plan)
    assert pf.permutation_pass_count() == 0


def test_filter_plan_binding(pf):
    """test_convolution.cpp:81-97."""
    plan = pf.Plan(2, [16])
    filt = pf.prepare_filter(rand_c(16, 79), plan)
    x = rand_c(16, 80)
    with pytest.raises(pf.FilterPlanMismatch):
        pf.convolve_permfree(x, filt, pf.Plan(4, [16]))
    with pytest.raises(RuntimeError):
        pf.convolve_permfree(x.reshape(4, 4), filt, pf.Plan(2, [4, 4]))
    pf.convolve_permfree(x, filt, pf.Plan(2, [16]))  # an equivalent plan is accepted
    with pytest.raises(pf.FilterPlanMismatch):
        pf.convolve_permfree(x, filt, pf.Plan(2, [16], precision=pf.F32))


def test_reuse_without_drift_bitwise(pf, torch):
    """test_convolution.cpp:99-111: repeated calls are bitwise identical."""
    plan = pf.Plan(2, [8, 8])
    filt = pf.prepare_filter(rand_c(64, 83).reshape(8, 8, order="F"), plan)
    x = rand_c(64, 84).reshape(8, 8, order="F")
    first = pf.convolve_permfree(x, filt, plan)
    for _ in range(3):
        assert np.array_equal(pf.convolve_permfree(x, filt, plan), first)
    # and on a large multi-pass plan, device path
    big = pf.Plan(3, [3 ** 13])
    gb = torch.from_numpy(rand_c(3 ** 13, 5)).cuda()
    fb = pf.prepare_filter_device(gb, big)
    xb = torch.from_numpy(rand_c(3 ** 13, 6)).cuda()
    y1 = pf.convolve_permfree_out(xb, torch.empty_like(xb), fb, big)
    y2 = pf.convolve_permfree_out(xb, torch.empty_like(xb), fb, big)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("radix,dims", [(2, [4096]), (4, [64, 64]), (8, [8, 64]), (2, [4, 2, 8]), (3, [2187]),
                                        (5, [25, 125]), (2, [1 << 16]), (3, [9, 243])])
def test_transforms_match_numpy(pf, radix, dims):
    """test_smoke.py:20-31 and test_butterfly.cpp:74-104 (ladder o reversal = DFT)."""
    rng = np.random.default_rng(1)
    shape = tuple(dims)
    a = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
    plan = pf.Plan(radix, dims)
    n = plan.total
    F = np.fft.fftn(a)
    tol = transform_tolerance(n, np.abs(a).max()) * max(1.0, np.sqrt(n) / 8)
    assert max_diff(pf.fft_forward(a, plan), F) <= max(tol, 1e-10)
    assert rel_l2(pf.fft_forward(a, plan), F) <= 1e-13
    assert rel_l2(pf.fft_backward(F, plan), a) <= 1e-13
    # A^T leaves P * F: permuting it back gives F
    assert rel_l2(pf.permute(pf.fft_transposed(a, plan), plan), F) <= 1e-13
    # unordered forward on reversed input == forward (test_smoke.py:54-59 shape)
    assert rel_l2(pf.fft_forward_unordered(pf.permute(a, plan), plan), F) <= 1e-13


def test_four_point_ladders_known_answers(pf):
    """test_butterfly.cpp:28-45."""
    plan = pf.Plan(2, [4])
    assert max_diff(pf.fft_forward_unordered(np.array([1, 3, 2, 4], dtype=complex), plan),
                    [10, -2 + 2j, -2, -2 - 2j]) < 1e-13
    y = pf.fft_backward_unordered(np.array([10, -2, -2 + 2j, -2 - 2j]), plan) * 4
    assert max_diff(y, [4, 8, 12, 16]) < 1e-13
    assert max_diff(pf.fft_transposed(np.array([1, 2, 3, 4], dtype=complex), plan),
                    [10, -2, -2 + 2j, -2 - 2j]) < 1e-13


def test_permutation_involution_bitwise(pf):
    """test_permutation.cpp:312-331."""
    for radix, dims in [(2, [64, 64]), (4, [64, 16]), (8, [4096]), (2, [16, 16, 16]), (3, [27, 9]), (5, [125])]:
        plan = pf.Plan(radix, dims)
        x = rand_c(plan.total, 23).reshape(dims, order="F")
        y = pf.permute(x, plan)
        assert np.array_equal(np.sort(y.real.ravel()), np.sort(x.real.ravel()))
        assert np.array_equal(pf.permute(y, plan), x)


def test_prepare_from_impulse_equals_reversed_spectrum(pf, torch, orc):
    for radix, dims in [(2, [1024]), (3, [729]), (4, [16, 64]), (5, [625]), (3, [3 ** 13])]:
        n = int(np.prod(dims))
        h = rand_c(n, 11)
        op = orc.plan(radix, dims)
        ghat_ref = op.prepare_filter(op.filter_from_impulse(h))
        plan = pf.Plan(radix, dims)
        f = pf.prepare_filter_from_impulse(torch.from_numpy(h).cuda(), plan)
        assert rel_l2(f.ghat, ghat_ref) <= 1e-13


def test_batched_and_out_of_place(pf, torch, orc):
    radix, dims, batch = 3, [729], 5
    n = 729
    xs = np.stack([rand_c(n, 100 + b) for b in range(batch)])
    h = rand_c(n, 99)
    op = orc.plan(radix, dims)
    ghat = op.prepare_filter(op.filter_from_impulse(h))
    ref = np.stack([op.convolve_permfree(xs[b], ghat) for b in range(batch)])
    plan = pf.Plan(radix, dims)
    f = pf.prepare_filter_from_impulse(torch.from_numpy(h).cuda(), plan)
    xt = torch.from_numpy(xs).cuda()
    x0 = xt.clone()
    y = pf.convolve_permfree_out(xt, torch.empty_like(xt), f, plan)
    torch.cuda.synchronize()
    assert torch.equal(xt, x0)  # input untouched
    assert rel_l2(y.cpu().numpy(), ref) <= 1e-12
    # host pipelined path
    hx = np.ascontiguousarray(xs.copy())
    pf.convolve_permfree_host(hx, f, plan)
    assert rel_l2(hx, ref) <= 1e-12


@pytest.mark.parametrize("mid,strided", [(3, 2), (4, 3), (2, 2)])
def test_forced_multipass_schedules(pf, torch, orc, mid, strided, monkeypatch):
    """Small shapes forced through many passes (strided DIF/DIT with external
    twiddles) to pin the large-n code paths at oracle-checkable sizes."""
    monkeypatch.setenv("PAFFT_MAX_MID_STAGES", str(mid))
    monkeypatch.setenv("PAFFT_MAX_STRIDED_STAGES", str(strided))
    for radix, dims in [(2, [4096]), (3, [2187]), (4, [1024]), (5, [3125]), (8, [4096]), (2, [64, 128]),
                        (3, [81, 27]), (4, [16, 64, 4])]:
        n = int(np.prod(dims))
        x, h = rand_c(n, 1), rand_c(n, 2)
        y_orc, g, _ = _oracle_conv(orc, radix, dims, x, h)
        plan = pf.Plan(radix, dims)
        if max(round(np.log(d) / np.log(radix)) for d in dims[:1]) > mid or len(dims) > 1:
            assert plan.num_passes() >= 3, plan.describe()
        f = pf.prepare_filter_device(torch.from_numpy(g).cuda(), plan)
        assert rel_l2(dev_conv(pf, torch, plan, f, x), y_orc) <= 1e-12, plan.describe()
        # fp32: the north star's 1e-5 bar against the fp64 pipeline on the
        # fp32-rounded inputs
        x32, g32 = x.astype(np.complex64), g.astype(np.complex64)
        op = orc.plan(radix, dims)
        y_orc32 = op.convolve_permfree(x32.astype(np.complex128), op.prepare_filter(g32.astype(np.complex128)))
        p32 = pf.Plan(radix, dims, precision=pf.F32)
        f32 = pf.prepare_filter_device(torch.from_numpy(g32).cuda(), p32)
        y32 = dev_conv(pf, torch, p32, f32, x32)
        assert rel_l2(y32, y_orc32) <= 1e-5, (radix, dims, rel_l2(y32, y_orc32), p32.describe())


def test_filter_key_includes_conv_slot_layout(pf, torch, orc, monkeypatch):
    """The kernel copy of ghat is stored in the CONV pass's slot order, which
    depends on the pass schedule (PAFFT_* tuning variables read at plan
    creation).  A filter prepared under one schedule must be rejected by an
    equal-shape plan built under another, and the spectrum cache must not hand
    one schedule's copy to the other."""
    radix, dims = 3, [2187]
    n = 2187
    x, h = rand_c(n, 5), rand_c(n, 6)
    y_orc, g, _ = _oracle_conv(orc, radix, dims, x, h)
    plan_a = pf.Plan(radix, dims)
    f_a = pf.prepare_filter_device(torch.from_numpy(g).cuda(), plan_a)
    monkeypatch.setenv("PAFFT_MAX_MID_STAGES", "3")
    monkeypatch.setenv("PAFFT_MAX_STRIDED_STAGES", "2")
    plan_b = pf.Plan(radix, dims)
    monkeypatch.delenv("PAFFT_MAX_MID_STAGES")
    monkeypatch.delenv("PAFFT_MAX_STRIDED_STAGES")
    assert plan_a.describe() != plan_b.describe()
    with pytest.raises(pf.FilterPlanMismatch):
        dev_conv(pf, torch, plan_b, f_a, x)
    ht = torch.from_numpy(h).cuda()
    c_a = pf.prepare_filter_from_impulse(ht, plan_a, cache=True)
    c_b = pf.prepare_filter_from_impulse(ht, plan_b, cache=True)
    assert rel_l2(dev_conv(pf, torch, plan_a, c_a, x), y_orc) <= 1e-12
    assert rel_l2(dev_conv(pf, torch, plan_b, c_b, x), y_orc) <= 1e-12
