"""Threading contract (SPEC.md:89/:220/:366, test_transform.cpp:141-155):
Plan and PreparedFilter are immutable and shareable; calls on distinct
buffers may run concurrently from several threads (here: each thread on its
own CUDA stream), and the permutation-pass counter is per thread.  Every
concurrent result must equal the single-threaded result bit for bit."""
import threading

import numpy as np
import pytest

from helpers import rand_c

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


@pytest.mark.parametrize("radix,dims", [(3, [2187]), (2, [64, 64]), (5, [625])])
def test_concurrent_calls_share_plan_and_filter(pf, torch, radix, dims):
    plan = pf.Plan(radix, dims)
    n = plan.total
    h = torch.from_numpy(rand_c(n, 1)).cuda()
    filt = pf.prepare_filter_from_impulse(h, plan)
    g = h.clone()
    pf.fft_forward_(g, plan)  # natural-order spectrum for the standard path
    nthreads, rounds = 4, 6
    inputs = [torch.from_numpy(np.stack([rand_c(n, 10 * t + b) for b in range(3)])).cuda() for t in range(nthreads)]
    host_in = [rand_c(n, 500 + t).reshape(dims) for t in range(nthreads)]
    hg = np.fft.fftn(rand_c(n, 2).reshape(dims))

    def work(t, x, hx):
        # permfree (device, out of place), standard (device, in place), forward
        # transform (device), permfree through the host split API
        y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan)
        ys = x.clone()
        pf.convolve_standard_(ys, g, plan)
        yf = x.clone()
        pf.fft_forward_(yf, plan)
        yh = pf.convolve_permfree(hx, pf.prepare_filter(hg, plan), plan)
        return y, ys, yf, yh

    torch.cuda.synchronize()
    want = []
    for t in range(nthreads):
        r = work(t, inputs[t], host_in[t])
        torch.cuda.synchronize()
        want.append([v.cpu().numpy() if hasattr(v, "cpu") else v for v in r])

    got = [None] * nthreads
    counts = [None] * nthreads
    errors = []

    def runner(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                pf.reset_permutation_pass_count()
                for _ in range(rounds):
                    r = work(t, inputs[t], host_in[t])
                s.synchronize()
                counts[t] = pf.permutation_pass_count()
                got[t] = [v.cpu().numpy() if hasattr(v, "cpu") else v for v in r]
        except Exception as e:  # surfaced below
            errors.append(e)

    ths = [threading.Thread(target=runner, args=(t,)) for t in range(nthreads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
    for t in range(nthreads):
        for a, b in zip(got[t], want[t]):
            assert np.array_equal(a, b)
    # per thread: 3 signals x (2 standard + 1 forward) permutations + 1 host
    # prepare_filter per round -- only this thread's calls
    assert counts == [rounds * (3 * 3 + 1)] * nthreads, counts
