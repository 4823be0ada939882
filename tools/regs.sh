#!/bin/bash
# Per-kernel registers/spills for one instance TU: tools/regs.sh r3_f64 [extra nvcc flags]
f=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xptxas -v --expt-relaxed-constexpr -Iinclude "$@" \
  -c paper_2506_12718_b200/csrc/inst/inst_$f.cu -o /tmp/regs_$f.o 2>&1 | python3 -c "
import sys,re
cur=None; sp=None
for line in sys.stdin:
    if 'error' in line: print(line)
    m=re.search(r\"Compiling entry function '_ZN10pafft_b20011pass_kernelI[df](\w+)'\",line)
    if m: cur=m.group(1); continue
    m2=re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads',line)
    if m2: sp=(int(m2.group(1)), int(m2.group(2)))
    m=re.search(r'Used (\d+) registers',line)
    if m and cur:
        a=re.findall(r'Li(\d+)E',cur); print('r%s R=%s kind=%s map=%s regs=%s spill=%s' % (a[0], 'x'.join(a[1:5]), a[5], a[6], m.group(1), sp)); cur=None
"
