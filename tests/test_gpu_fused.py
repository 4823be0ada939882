"""The opt-in fused single-launch convolution (PAFFT_FUSED=1, csrc/fused.cuh).

It runs the same tile bodies as the three-launch path, so its results must be
bitwise identical to it; checked at the 1-D BASELINE shapes it is compiled for
(configs 1, 2, 5), with small and ragged batches, several lags (pipeline depth
between the passes) and in place.  Measured on B200 it is slower than the
three launches, which is why it stays opt-in.
"""
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2506_12718_b200 as pf
    from paper_2506_12718_b200 import workload
    assert torch.cuda.is_available()
    yield pf, torch, workload
    os.environ.pop("PAFFT_FUSED", None)
    os.environ.pop("PAFFT_FUSED_LAG", None)


def _run(pf, torch, plan, filt, x, fused, lag=None, inplace=False):
    os.environ["PAFFT_FUSED"] = "1" if fused else "0"
    if lag is None:
        os.environ.pop("PAFFT_FUSED_LAG", None)
    else:
        os.environ["PAFFT_FUSED_LAG"] = str(lag)
    if inplace:
        y = x.clone()
        pf.convolve_permfree_(y, filt, plan)
    else:
        y = torch.empty_like(x)
        pf.convolve_permfree_out(x, y, filt, plan)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("idx,batch,lag", [(2, 1, None), (2, 3, None), (2, 5, 2), (5, 1, None), (5, 37, None),
                                           (5, 64, 1), (5, 64, 64), (1, 1, None), (1, 3, 1)])
def test_fused_bitwise_equals_three_launches(env, idx, batch, lag):
    pf, torch, workload = env
    cfg = workload.get_config(idx, "f64")
    plan = pf.Plan(cfg.radix, cfg.dims, precision=pf.F64)
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(workload.impulse(cfg)).to("cuda", torch.complex128), plan)
    xs = workload.signals(cfg, 0, batch)
    x = torch.from_numpy(xs).to("cuda", torch.complex128).reshape(batch, -1)
    n0 = pf.lib.pafft_kernel_launch_count()
    y3 = _run(pf, torch, plan, filt, x, fused=False)
    n1 = pf.lib.pafft_kernel_launch_count()
    yf = _run(pf, torch, plan, filt, x, fused=True, lag=lag)
    n2 = pf.lib.pafft_kernel_launch_count()
    assert n1 - n0 == 3 and n2 - n1 == 1, "fused path must be one launch"
    assert torch.equal(y3, yf)
    yi = _run(pf, torch, plan, filt, x, fused=True, lag=lag, inplace=True)
    assert torch.equal(y3, yi)
