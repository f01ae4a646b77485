#!/bin/bash
set -u
O=gpurun_out/r2s; mkdir -p $O
for v in r64m6 r64w128m5; do
  CLB_LIB_VARIANT=$v timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or sw2048 or segmentation" > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
done
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 sw8192 sw8192hump sw8192f32 c5 c5f32; do
  for v in r64m6 r64w128m5; do
    CLB_LIB_VARIANT=$v b $w ${w}_$v
  done
done
echo done > $O/DONE
