#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for w in sw8192f32 c5 c5f32 c3; do
  for v in tma shfl; do
    CLB_CONTIG=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > $O/bench_${w}_$v.json 2>&1
  done
done
