#!/bin/bash
set -u
O=gpurun_out/r2m; mkdir -p $O
CLB_LIB_VARIANT=x2 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or c5 or c4 or segmentation or hump" > $O/pytest_x2.log 2>&1; echo "pytest rc=$?" >> $O/pytest_x2.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c5 c5f32 c4 sw8192 sw8192hump sw8192f32; do
  b $w ${w}_base
  CLB_LIB_VARIANT=x2 b $w ${w}_x2
done
echo done > $O/DONE
