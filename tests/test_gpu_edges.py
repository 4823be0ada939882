"""Edge cases and maximum sizes on the GPU: extent-1 axes, empty batches,
device buffers the kernels cannot stage (fp32 pointers off a 16-byte
boundary) and launch-size limits fail cleanly, and the largest practical
plans (2^27, 3^17, 5^11 points, 8192^2, 512^3) pass size-independent
properties on device: delta -> identity, shifted delta -> cyclic shift,
linearity."""
import ctypes as C

import numpy as np
import pytest

from helpers import rand_c, rel_l2

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


@pytest.mark.parametrize("radix,dims", [(2, [1]), (3, [1, 27]), (2, [16, 1]), (5, [1, 1, 25]), (4, [1, 4, 1])],
                         ids=lambda v: str(v))
def test_extent_one_axes(pf, torch, orc, radix, dims):
    n = int(np.prod(dims))
    x, h = rand_c(n, 1), rand_c(n, 2)
    plan = pf.Plan(radix, dims)
    f = pf.prepare_filter_from_impulse(torch.from_numpy(h).cuda(), plan)
    y = pf.convolve_permfree_out(torch.from_numpy(x).cuda(), torch.empty(n, dtype=torch.complex128, device="cuda"),
                                 f, plan).cpu().numpy()
    shp = dims[::-1]
    want = np.fft.ifftn(np.fft.fftn(x.reshape(shp)) * np.fft.fftn(h.reshape(shp))).reshape(-1)
    assert rel_l2(y, want) <= 1e-13
    op = orc.plan(radix, dims)
    assert rel_l2(y, op.convolve_permfree(x, op.prepare_filter(op.filter_from_impulse(h)))) <= 1e-13


def test_empty_batch_is_a_no_op(pf, torch):
    plan = pf.Plan(3, [243])
    f = pf.prepare_filter_from_impulse(torch.from_numpy(rand_c(243, 1)).cuda(), plan)
    x = torch.empty(0, 243, dtype=torch.complex128, device="cuda")
    pf.convolve_permfree_(x, f, plan)
    pf.convolve_permfree_out(x, torch.empty_like(x), f, plan)
    torch.cuda.synchronize()


def test_unstageable_buffers_fail_cleanly(pf, torch):
    """fp32 device pointers 8 bytes off a 16-byte boundary cannot feed TMA:
    a clean error, never a wrong answer."""
    plan = pf.Plan(3, [2187], precision=pf.F32)
    f = pf.prepare_filter_from_impulse(torch.from_numpy(rand_c(2187, 1)).to("cuda", torch.complex64), plan)
    base = torch.from_numpy(rand_c(2 * 2187 + 1, 2)).to("cuda", torch.complex64)
    x = base[1:2188]
    assert x.data_ptr() % 16 == 8
    with pytest.raises(RuntimeError):
        pf.convolve_permfree_out(x, torch.empty(2187, dtype=torch.complex64, device="cuda"), f, plan)
    # aligned views of the same storage work
    xa = base[2:2189]
    assert xa.data_ptr() % 16 == 0
    y = pf.convolve_permfree_out(xa, torch.empty(2187, dtype=torch.complex64, device="cuda"), f, plan)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(y)).all()


def test_launch_size_limit_is_reported(pf):
    """More than 2^31 tiles in one call: INVALID_ARGUMENT before any memory
    is touched (the caller splits the batch)."""
    from paper_2506_12718_b200 import _lib
    plan = pf.Plan(2, [2])
    f = pf.empty_filter(plan)
    st = _lib.lib.pafft_convolve_permfree_oop(plan._h, f._h, C.c_void_p(0x10000), C.c_void_p(0x20000),
                                              C.c_size_t(2 ** 31 + 5), None)
    assert st == 7  # PAFFT_INVALID_ARGUMENT


@pytest.mark.parametrize("radix,dims", [(2, [1 << 27]), (3, [3 ** 17]), (5, [5 ** 11]), (2, [8192, 8192]),
                                        (2, [512, 512, 512]), (3, [3 ** 8, 3 ** 7])],
                         ids=lambda v: str(v))
def test_maximum_sizes_properties(pf, torch, radix, dims):
    n = int(np.prod(dims))
    plan = pf.Plan(radix, dims)
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.complex(torch.rand(n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1,
                      torch.rand(n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1)
    # delta -> identity
    d = torch.zeros(n, dtype=torch.complex128, device="cuda")
    d[0] = 1
    y = pf.convolve_permfree_out(x, torch.empty_like(x), pf.prepare_filter_from_impulse(d, plan), plan)
    assert float(torch.linalg.vector_norm(y - x) / torch.linalg.vector_norm(x)) <= 1e-13
    # shifted delta -> cyclic shift along axis 0 (and axis 1 for multi-dim)
    s0 = 3
    idx = s0 + (dims[0] * 2 if len(dims) > 1 else 0)
    d.zero_()
    d[idx] = 1
    y = pf.convolve_permfree_out(x, y, pf.prepare_filter_from_impulse(d, plan), plan)
    xs = x.view(*dims[::-1])
    want = torch.roll(xs, shifts=s0, dims=len(dims) - 1)
    if len(dims) > 1:
        want = torch.roll(want, shifts=2, dims=len(dims) - 2)
    assert float(torch.linalg.vector_norm(y - want.reshape(-1)) / torch.linalg.vector_norm(x)) <= 1e-13
    del want, xs
    # linearity with a random filter
    h = torch.complex(torch.randn(n, device="cuda", dtype=torch.float64, generator=g),
                      torch.randn(n, device="cuda", dtype=torch.float64, generator=g))
    f = pf.prepare_filter_from_impulse(h, plan)
    x2 = torch.flip(x, dims=[0])
    a, b = 0.75 - 0.5j, -1.25 + 0.25j
    lhs = pf.convolve_permfree_out(a * x + b * x2, torch.empty_like(x), f, plan)
    r1 = pf.convolve_permfree_out(x, torch.empty_like(x), f, plan)
    r2 = pf.convolve_permfree_out(x2, x2, f, plan)  # in place
    torch.cuda.synchronize()
    assert float(torch.linalg.vector_norm(lhs - (a * r1 + b * r2)) / torch.linalg.vector_norm(lhs)) <= 1e-12


@pytest.mark.parametrize("radix,dims,batch", [(4, [256, 256, 16], 2), (2, [64, 256, 8], 4), (8, [8, 64, 64], 3)])
def test_wide_strided_tiles_are_bitwise_the_narrow_ones(pf, torch, monkeypatch, radix, dims, batch):
    """Launches with many tiles take the 16-column strided instances
    (inst_wide.cu, use_wide); per column they do the same arithmetic as the
    8-column ones, so the convolution is bitwise identical (PAFFT_WIDE=0 at
    plan creation disables them)."""
    import numpy as np
    n = int(np.prod(dims))
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).cuda()
    h = torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n)).cuda()
    wide = pf.Plan(radix, dims)
    monkeypatch.setenv("PAFFT_WIDE", "0")
    narrow = pf.Plan(radix, dims)
    monkeypatch.delenv("PAFFT_WIDE")
    assert "many tiles" in wide.describe() and "many tiles" not in narrow.describe()
    yw = pf.convolve_permfree_out(x, torch.empty_like(x), pf.prepare_filter_from_impulse(h, wide), wide)
    yn = pf.convolve_permfree_out(x, torch.empty_like(x), pf.prepare_filter_from_impulse(h, narrow), narrow)
    torch.cuda.synchronize()
    assert torch.equal(yw, yn)


@pytest.mark.parametrize("radix,dims,batch", [(2, [64, 256, 8], 3), (4, [256, 64], 5), (8, [64, 512], 2),
                                              (2, [4096, 32], 4)])
def test_fp32_dense_strided_tiles_are_bitwise_the_spare_slot_ones(pf, torch, monkeypatch, radix, dims, batch):
    """fp32 strided tiles of even row length take the dense instance (tensor-map
    staging and stores, no spare row slots; pafft_b200.cu make_pass); per column
    it does the same arithmetic as the spare-slot instance that odd row lengths
    need, so the convolution is bitwise identical (PAFFT_F32_DENSE=0 at plan
    creation disables it)."""
    n = int(np.prod(dims))
    rng = np.random.default_rng(17)
    x = torch.from_numpy((rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).astype(np.complex64)).cuda()
    h = torch.from_numpy((rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)).cuda()
    dense = pf.Plan(radix, dims, precision=pf.F32)
    monkeypatch.setenv("PAFFT_F32_DENSE", "0")
    spare = pf.Plan(radix, dims, precision=pf.F32)
    monkeypatch.delenv("PAFFT_F32_DENSE")
    assert dense.num_passes() == spare.num_passes() >= 3
    yd = pf.convolve_permfree_out(x, torch.empty_like(x), pf.prepare_filter_from_impulse(h, dense), dense)
    ys = pf.convolve_permfree_out(x, torch.empty_like(x), pf.prepare_filter_from_impulse(h, spare), spare)
    torch.cuda.synchronize()
    assert torch.equal(yd, ys)


def test_fp32_odd_row_lengths_take_short_strided_groups(pf, torch, orc, monkeypatch):
    """fp32 axes whose strided rows have an odd number of elements stop at 81
    (radix 3) / 125 (radix 5) rows per strided pass (build_groups): 3^12 runs
    DIF 9, DIF 27, CONV 3^7, DIT 27, DIT 9 instead of DIF 243, CONV, DIT 243;
    both schedules meet the fp32 bar against the fp64 pipeline on the rounded
    inputs."""
    dims = [3 ** 12]
    n = dims[0]
    x32 = rand_c(n, 3).astype(np.complex64)
    h32 = rand_c(n, 4).astype(np.complex64)
    op = orc.plan(3, dims)
    want = op.convolve_permfree(x32.astype(np.complex128),
                                op.prepare_filter(op.filter_from_impulse(h32.astype(np.complex128))))
    short = pf.Plan(3, dims, precision=pf.F32)
    monkeypatch.setenv("PAFFT_F32_ODD_SINGLE", "0")
    long_ = pf.Plan(3, dims, precision=pf.F32)
    monkeypatch.delenv("PAFFT_F32_ODD_SINGLE")
    assert short.num_passes() == 5 and long_.num_passes() == 3, (short.describe(), long_.describe())
    for plan in (short, long_):
        xt = torch.from_numpy(x32).cuda()
        f = pf.prepare_filter_from_impulse(torch.from_numpy(h32).cuda(), plan)
        pf.convolve_permfree_(xt, f, plan)
        torch.cuda.synchronize()
        assert rel_l2(xt.cpu().numpy().astype(np.complex128), want) <= 1e-5, plan.describe()
    # fp64 plans are not affected
    assert pf.Plan(3, dims).num_passes() == 3
