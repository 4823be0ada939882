"""Multi-GPU filter distribution through the C ABI (pafft_filter_broadcast,
SURVEY.md 8b/8e): NCCL broadcast of a prepared filter, once per filter.  The
round-end box has one GPU, so the single-device call (NCCL load, clique
creation, in-place broadcast, receiver rebuild) and the error contract run
everywhere; the cross-device copy runs when >= 2 GPUs are visible."""
import numpy as np
import pytest

from helpers import rel_l2

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


def _filter(pf, torch, plan, seed=7, device=0):
    rng = np.random.default_rng(seed)
    h = rng.standard_normal(plan.total) + 1j * rng.standard_normal(plan.total)
    return h, pf.prepare_filter_from_impulse(torch.from_numpy(h).to(f"cuda:{device}"), plan)


def test_single_device_broadcast_keeps_filter(pf, torch, orc):
    plan = pf.Plan(3, [2187])
    h, f = _filter(pf, torch, plan)
    before = pf.filter_device_tensor(f).clone()
    before_k = pf.filter_device_tensor(f, scaled=True).clone()
    pf.broadcast_filter_nccl([f], root=0)
    torch.cuda.synchronize()
    assert torch.equal(pf.filter_device_tensor(f), before)
    assert torch.equal(pf.filter_device_tensor(f, scaled=True), before_k)
    x = np.random.default_rng(1).uniform(-1, 1, (2, plan.total * 2)).view(np.complex128)
    xt = torch.from_numpy(x).cuda()
    y = pf.convolve_permfree_out(xt, torch.empty_like(xt), f, plan).cpu().numpy()
    op = orc.plan(3, [2187])
    gh = op.prepare_filter(op.filter_from_impulse(h))
    for b in range(2):
        assert rel_l2(y[b], op.convolve_permfree(x[b], gh)) <= 1e-12


def test_broadcast_error_contract(pf, torch):
    plan = pf.Plan(3, [729])
    _, f = _filter(pf, torch, plan)
    other = pf.empty_filter(pf.Plan(3, [243]))
    with pytest.raises(pf.FilterPlanMismatch):
        pf.broadcast_filter_nccl([f, other])
    same_dev = pf.empty_filter(plan)
    with pytest.raises(RuntimeError):
        pf.broadcast_filter_nccl([f, same_dev])  # one filter per device
    with pytest.raises(RuntimeError):
        pf.broadcast_filter_nccl([f], root=3)


def test_two_device_broadcast(pf, torch, orc):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    p0 = pf.Plan(5, [3125], device=0)
    p1 = pf.Plan(5, [3125], device=1)
    h, f0 = _filter(pf, torch, p0)
    f1 = pf.empty_filter(p1)
    pf.broadcast_filter_nccl([f0, f1], root=0)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    assert torch.equal(pf.filter_device_tensor(f1).cpu(), pf.filter_device_tensor(f0).cpu())
    x = np.random.default_rng(2).uniform(-1, 1, p0.total * 2).view(np.complex128)
    y0 = pf.convolve_permfree_out(torch.from_numpy(x).to("cuda:0"), torch.empty(p0.total, dtype=torch.complex128,
                                  device="cuda:0"), f0, p0).cpu()
    y1 = pf.convolve_permfree_out(torch.from_numpy(x).to("cuda:1"), torch.empty(p1.total, dtype=torch.complex128,
                                  device="cuda:1"), f1, p1).cpu()
    assert torch.equal(y0, y1)


def test_filter_spectrum_cache_across_plans(pf, torch):
    """a spectrum prepared from the same impulse for a
    plan with the same key is shared, not recomputed; held weakly."""
    import gc
    p1, p2 = pf.Plan(3, [2187]), pf.Plan(3, [2187])
    rng = np.random.default_rng(11)
    h = torch.from_numpy(rng.standard_normal(2187) + 1j * rng.standard_normal(2187)).cuda()
    h0, m0, _ = pf.filter_cache_stats()
    f1 = pf.prepare_filter_from_impulse(h, p1, cache=True)
    f2 = pf.prepare_filter_from_impulse(h, p2, cache=True)
    assert not f1.cache_hit and f2.cache_hit
    assert f1.device_ghat_ptr(True) == f2.device_ghat_ptr(True)
    ref = pf.prepare_filter_from_impulse(h, p2)  # uncached: same bits
    assert torch.equal(pf.filter_device_tensor(f2), pf.filter_device_tensor(ref))
    x = torch.from_numpy(rng.uniform(-1, 1, (2, 2187)) + 0j).cuda()
    y1 = pf.convolve_permfree_out(x, torch.empty_like(x), f1, p1)
    y2 = pf.convolve_permfree_out(x, torch.empty_like(x), f2, p2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    # other bytes, other key -> misses
    g = h.clone()
    g[5] += 1.0
    assert not pf.prepare_filter_from_impulse(g, p1, cache=True).cache_hit
    assert not pf.prepare_filter_from_impulse(h.to(torch.complex64), pf.Plan(3, [2187], precision=pf.F32),
                                              cache=True).cache_hit
    hits, misses, _ = pf.filter_cache_stats()
    assert hits - h0 >= 1 and misses - m0 >= 3
    # weak entries: once every handle is gone the spectrum is released
    del f1, f2
    gc.collect()
    assert not pf.prepare_filter_from_impulse(h, p1, cache=True).cache_hit
