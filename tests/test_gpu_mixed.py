"""Per-axis radices on the GPU:
plans whose axes are powers of different radices, e.g. 3^3 x 2^6.  Each axis
runs its own radix's pass kernels and the prepared filter is the per-axis
digit reversal.  Checked against the oracle's mixed plans (pinned in
tests/test_oracle_pins.py::test_mixed_radix_oracle_pins) on the same inputs."""
import numpy as np
import pytest

from helpers import GRID_MIXED, rand_c, rel_l2

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


def _run(pf, torch, orc, radices, dims, prec, batch=2):
    n = int(np.prod(dims))
    cdt = torch.complex128 if prec == pf.F64 else torch.complex64
    xs = np.stack([rand_c(n, 100 + b) for b in range(batch)])
    h = rand_c(n, 99)
    if prec == pf.F32:
        xs = xs.astype(np.complex64).astype(np.complex128)
        h = h.astype(np.complex64).astype(np.complex128)
    plan = pf.Plan(radices, dims, precision=prec)
    f = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    x = torch.from_numpy(xs).to("cuda", cdt)
    y = pf.convolve_permfree_out(x, torch.empty_like(x), f, plan).cpu().numpy().astype(np.complex128)
    op = orc.plan(list(radices), dims)
    gh = op.prepare_filter(op.filter_from_impulse(h))
    return [rel_l2(y[b], op.convolve_permfree(xs[b], gh)) for b in range(batch)]


@pytest.mark.parametrize("radices,dims", GRID_MIXED, ids=lambda v: str(v))
def test_mixed_permfree_matches_oracle(pf, torch, orc, radices, dims):
    assert max(_run(pf, torch, orc, radices, dims, pf.F64)) <= 1e-12


@pytest.mark.parametrize("radices,dims", [([3, 2], [27, 64]), ([5, 4], [25, 64]), ([2, 3, 5], [8, 9, 25])],
                         ids=lambda v: str(v))
def test_mixed_permfree_fp32(pf, torch, orc, radices, dims):
    assert max(_run(pf, torch, orc, radices, dims, pf.F32)) <= 1e-5


@pytest.mark.parametrize("radices,dims", [([3, 2], [3 ** 9, 128]), ([2, 5], [4096, 625]), ([4, 3], [4096, 729])],
                         ids=lambda v: str(v))
def test_mixed_multipass_against_numpy(pf, torch, radices, dims):
    """Axes long enough for multi-stage passes on both radices (CONV pass of
    axis 0's radix, strided passes of the other)."""
    n = int(np.prod(dims))
    plan = pf.Plan(radices, dims)
    assert plan.radices == list(radices) and plan.num_passes() >= 3
    x, h = rand_c(n, 5), rand_c(n, 6)
    f = pf.prepare_filter_from_impulse(torch.from_numpy(h).cuda(), plan)
    y = pf.convolve_permfree_out(torch.from_numpy(x[None]).cuda(), torch.empty(1, n, dtype=torch.complex128,
                                 device="cuda"), f, plan).cpu().numpy()[0]
    shp = dims[::-1]
    want = np.fft.ifftn(np.fft.fftn(x.reshape(shp)) * np.fft.fftn(h.reshape(shp))).reshape(-1)
    assert rel_l2(y, want) <= 1e-12


def test_mixed_prepare_filter_bit_exact_and_transforms(pf, torch, orc):
    radices, dims = [3, 4], [81, 64]
    n = int(np.prod(dims))
    g = rand_c(n, 3)
    plan = pf.Plan(radices, dims)
    op = orc.plan(radices, dims)
    # observable ghat: the per-axis digit reversal of g, bit for bit
    f = pf.prepare_filter_device(torch.from_numpy(g).cuda(), plan)
    assert np.array_equal(pf.filter_device_tensor(f).cpu().numpy(), op.prepare_filter(g))
    # transforms: natural-order DFT and the unordered ladders
    t = torch.from_numpy(g.copy()).cuda()
    pf.fft_forward_(t, plan)
    shp = dims[::-1]
    assert rel_l2(t.cpu().numpy(), np.fft.fftn(g.reshape(shp)).reshape(-1)) <= 1e-13
    # standard-order comparator equals the permutation-free path
    x = rand_c(n, 4)
    ys = torch.from_numpy(x.copy()).cuda()
    gs = torch.from_numpy(op.filter_from_impulse(rand_c(n, 8))).cuda()
    fh = pf.prepare_filter_device(gs, plan)
    pf.convolve_standard_(ys, gs, plan)
    yp = pf.convolve_permfree_out(torch.from_numpy(x).cuda(), torch.empty(n, dtype=torch.complex128, device="cuda"),
                                  fh, plan)
    torch.cuda.synchronize()
    assert rel_l2(ys.cpu().numpy(), yp.cpu().numpy()) <= 1e-13


def test_mixed_plan_validation_and_binding(pf, torch):
    with pytest.raises(pf.NotAPowerOfRadix) as e:
        pf.Plan([3, 2], [27, 27])
    assert (e.value.dim, e.value.extent) == (1, 27)
    with pytest.raises(RuntimeError):
        pf.Plan([3, 7], [27, 49])
    with pytest.raises(RuntimeError):
        pf.Plan([3], [27, 27])
    # 16 is a power of 2 and of 4: same dims, different radices -> different keys
    p24, p42, p2 = pf.Plan([2, 4], [16, 16]), pf.Plan([4, 2], [16, 16]), pf.Plan(2, [16, 16])
    assert p24.key() != p42.key() != p2.key()
    f = pf.prepare_filter_from_impulse(torch.from_numpy(rand_c(256, 1)).cuda(), p24)
    x = torch.from_numpy(rand_c(256, 2)).cuda()
    for other in (p42, p2):
        with pytest.raises(pf.FilterPlanMismatch):
            pf.convolve_permfree_(x, f, other)
    # all radices equal == the uniform plan, bitwise
    pm, pu = pf.Plan([3, 3], [27, 81]), pf.Plan(3, [27, 81])
    h = torch.from_numpy(rand_c(27 * 81, 3)).cuda()
    xa = torch.from_numpy(rand_c(27 * 81, 4)).cuda()
    ya = pf.convolve_permfree_out(xa, torch.empty_like(xa), pf.prepare_filter_from_impulse(h, pm), pm)
    yb = pf.convolve_permfree_out(xa, torch.empty_like(xa), pf.prepare_filter_from_impulse(h, pu), pu)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
