#!/bin/bash
# Register/stack use of the SW fp64 MC sweep kernels (x TMA, y strided) under
# extra defines: scripts/probe.sh [-DKNOB=V ...]   (fast: two kernels only)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -w \
  -DCLB_DEFAULT_LIB=1 -I paper_1805_08846_b200/csrc "$@" -c /tmp/probe/probe.cu -o /tmp/probe/probe.o || exit 1
cuobjdump -res-usage /tmp/probe/probe.o 2>&1 | grep -A1 "sweep_kernel" | grep REG | awk '{print $1, $2}'
cuobjdump -sass /tmp/probe/probe.o | awk '/Function :/{f=$3} /LDL|STL/{c[f]++} END{for(k in c) print substr(k,1,60), c[k]}'
