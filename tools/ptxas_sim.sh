#!/bin/bash
# registers / spills of every sim_kernel instantiation (template flags
# WRITE SCREEN64 WONLY EXACT COUNT ERR4): tools/ptxas_sim.sh [extra nvcc flags]
cd "$(dirname "$0")/../paper_2208_14567_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I../../include --expt-relaxed-constexpr \
  -Xptxas -v "$@" -c sim.cu -o /tmp/sim_ptxas.o 2>&1 | python3 -c "
import re, sys
txt = sys.stdin.read()
for m in re.finditer(r\"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers\", txt):
    name = m.group(1)
    k = re.search(r'sim_kernelILb(\d)ELb(\d)ELb(\d)ELb(\d)ELb(\d)ELb(\d)', name)
    if k: print(''.join(k.groups()), 'stack', m.group(2), 'spill st/ld', m.group(3), m.group(4), 'regs', m.group(5))
if 'error' in txt: print(txt[-3000:])
"
