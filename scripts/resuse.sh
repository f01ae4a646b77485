#!/bin/bash
# Compile one instantiation unit with extra defines and print register /
# stack use of its sweep kernels.  Usage: scripts/resuse.sh FAMILY DTYPE [-DKNOB=V ...]
FAM=$1; DT=$2; shift 2
OUT=/tmp/resuse_${FAM}_${DT}_$$.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -DCLB_DEFAULT_LIB=1 -DCLB_DTYPE=$DT -w "$@" -c paper_1805_08846_b200/csrc/clb_inst_${FAM}.cu -o $OUT || exit 1
cuobjdump -res-usage $OUT 2>&1 | grep -A1 "sweep_kernel\|sweep_contig" | grep -v "^--" | paste - - | \
  sed -E 's/.*Function _ZN3clb1[0-9](sweep_[a-z]+)I[df]NS_[0-9]+([A-Za-z]+)I[df]L?i?([0-9]*)[^E]*E+L?i?n?([0-9]+)ELb([01])(ELb([01]))?.*REG:([0-9]+) STACK:([0-9]+).*/\1 \2 N\3 lim\4 lit\5 contig\7 REG \8 STACK \9/' | sort | uniq
rm -f $OUT
