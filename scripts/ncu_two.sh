#!/bin/bash
# ncu --set full of one x-sweep and one y-sweep launch of a workload: TAG WORKLOAD
O=gpurun_out/$1; W=$2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|sweep_contig" -s 6 -c 2 \
  -o $O/prof_${W} python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $O/ncu_$W.log 2>&1
