#!/bin/bash
# x-sweep variant experiment: TMA-transpose vs warp-shuffle kernels per workload
O=gpurun_out/$1; mkdir -p $O
for w in c5 c5f32 sw8192f32 c3; do
  for v in tma shfl; do
    CLB_CONTIG=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > $O/bench_${w}_$v.json 2>&1
  done
done
echo done > $O/DONE
