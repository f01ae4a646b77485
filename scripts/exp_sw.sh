#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for w in sw8192 c4; do for v in tma shfl; do
  CLB_CONTIG=$v timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > $O/bench_${w}_${v}.json 2>&1
done; done
echo done > $O/DONE
