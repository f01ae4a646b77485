#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for w in c1 c2 c3; do
  for m in 32 24 16 12 8; do
    CLB_MIN_SEG=$m timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_seg$m.json 2>&1
  done
done
echo done > $O/DONE
