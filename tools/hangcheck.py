"""Run each (radix, dims, precision) permfree case in its own subprocess with a
short timeout, so a hanging kernel is identified without burning the GPU
budget.  Usage: python tools/hangcheck.py [timeout_s]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2506_12718_b200 as pf, oracle
radix, dims, prec = %r, %r, %r
n = int(np.prod(dims)); rng = np.random.default_rng(1)
x = rng.uniform(-1,1,n)+1j*rng.uniform(-1,1,n); h = rng.uniform(-1,1,n)+1j*rng.uniform(-1,1,n)
O = oracle.Oracle(); op = O.plan(radix, dims); g = op.filter_from_impulse(h)
want = op.convolve_permfree(x, op.prepare_filter(g))
plan = pf.Plan(radix, dims, precision=prec)
cdt = torch.complex128 if prec == 0 else torch.complex64
f = pf.prepare_filter_device(torch.from_numpy(g).to('cuda', cdt), plan)
xt = torch.from_numpy(x).to('cuda', cdt)
pf.convolve_permfree_(xt, f, plan); torch.cuda.synchronize()
print('%%.2e' %% oracle.rel_l2(xt.cpu().numpy().astype(complex), want), plan.describe().replace(chr(10), ' | '))
'''
cases = []
for r, ks in [(2, [13, 16]), (3, [8, 9]), (4, [7]), (5, [6]), (8, [5])]:
    for k in ks:
        cases.append((r, [r ** k]))
cases += [(2, [64, 128]), (3, [81, 27]), (4, [16, 64, 4]), (3, [243, 27]), (5, [125, 25])]
to = float(sys.argv[1]) if len(sys.argv) > 1 else 30
for prec in (0, 1):
    for r, d in cases:
        try:
            out = subprocess.run([sys.executable, "-c", CASE % (ROOT, r, d, prec)], capture_output=True, text=True,
                                 timeout=to)
            errs = [l for l in out.stderr.splitlines() if 'Error' in l]
            msg = out.stdout.strip() or (errs[0] if errs else out.stderr.strip()[-300:])
        except subprocess.TimeoutExpired:
            msg = "HANG (timeout)"
        print(f"prec={prec} r={r} dims={d}: {msg}", flush=True)
