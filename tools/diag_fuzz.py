import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2506_12718_b200 as pf, oracle
from helpers import rand_c, rel_l2
orc = oracle.Oracle()
def run(radices, dims, batch, f32, mid, oop=True):
    n = int(np.prod(dims)); prec = pf.F32 if f32 else pf.F64; cdt = torch.complex64 if f32 else torch.complex128
    xs = np.stack([rand_c(n, 7*n+b) for b in range(batch)]); h = rand_c(n, 3*n+1)
    if f32: xs = xs.astype(np.complex64).astype(np.complex128); h = h.astype(np.complex64).astype(np.complex128)
    if mid: os.environ["PAFFT_MID_STAGES"] = str(mid)
    plan = pf.Plan(radices, dims, precision=prec); os.environ.pop("PAFFT_MID_STAGES", None)
    op = orc.plan(list(radices), dims); g = op.filter_from_impulse(h)
    want = [op.convolve_permfree(xs[b], op.prepare_filter(g)) for b in range(batch)]
    filt = pf.prepare_filter_from_impulse(torch.from_numpy(h).to("cuda", cdt), plan)
    x = torch.from_numpy(xs).to("cuda", cdt)
    y = pf.convolve_permfree_out(x, torch.empty_like(x), filt, plan).cpu().numpy().astype(np.complex128)
    e = [rel_l2(y[b], want[b]) for b in range(batch)]
    print(radices, dims, batch, 'f32' if f32 else 'f64', mid, ['%.1e' % v for v in e], plan.describe().replace('\n', ' | '))
for args in [([2,4],[1,16],2,True,3), ([2,4],[1,16],2,False,3), ([2,4],[1,16],1,True,0), ([2,4],[1,16],2,True,0),
             ([4],[16],2,True,0), ([2,4],[1,16],3,True,0), ([2,4],[1,16],4,True,0), ([4],[16],3,True,0), ([4],[4],3,True,0),
             ([2],[8],3,True,0), ([3],[27],3,True,0), ([2],[32],3,True,0)]:
    run(*args)
