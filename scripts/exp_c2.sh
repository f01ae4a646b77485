#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for v in tma shfl; do for m in 8 12 16 24; do
  CLB_CONTIG=$v CLB_MIN_SEG=$m timeout 300 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu > $O/bench_c2_${v}_$m.json 2>&1
done; done
echo done > $O/DONE
