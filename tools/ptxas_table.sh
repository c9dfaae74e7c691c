#!/bin/bash
# registers / spills per unet_tc_kernel instantiation: tools/ptxas_table.sh [conv_tc.cu]
SRC=${1:-paper_2410_16727_b200/csrc/conv_tc.cu}
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -diag-suppress 128,177 -I include -I paper_2410_16727_b200/csrc -Xptxas -v -c $SRC -o /tmp/ptxas_tab.o 2>&1 | \
  python3 -c "
import re,sys
cur=None
for l in sys.stdin:
    m=re.search(r'Compiling entry function \'(_ZN2ps14unet_tc_kernel\w+)\'',l)
    if m: cur=re.findall(r'L[ib](\d+)E',m.group(1)); continue
    if cur and 'spill' in l: sp=re.findall(r'(\d+) bytes spill',l)
    if cur and 'Used' in l:
        r=re.search(r'Used (\d+) registers',l).group(1); print('<'+','.join(cur)+'>', 'regs',r,'spill',sp); cur=None
"
