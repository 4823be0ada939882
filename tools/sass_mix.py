"""Aggregate an ncu --page source --print-source sass CSV by opcode (dynamic counts)
and by stall reason.  Usage: python tools/sass_mix.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
tot = tots = 0
for r in rows[hi + 1:]:
    if len(r) <= ei:
        continue
    try:
        n = float(r[ei]); s = float(r[st])
    except ValueError:
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    cnt[o] += n; tot += n
    stall[o] += s; tots += s
for o, n in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {n / tot * 100:6.2f}% inst  {stall[o] / max(tots, 1) * 100:6.2f}% stall-samples")
print("total warp instructions", tot)
