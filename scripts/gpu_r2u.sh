#!/bin/bash
set -u
O=gpurun_out/r2u; mkdir -p $O
CLB_LIB_VARIANT=yinl3 timeout 1200 python -m pytest tests -m gpu -x -q -k "golden or random_configs or slow_path or segmentation or hump or c2_ or c4 or c3 or slab or blowup" > $O/pytest_yinl3.log 2>&1; echo "pytest rc=$?" >> $O/pytest_yinl3.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 sw8192 sw8192hump sw8192f32 c5 c5f32 c3 c2; do
  b $w ${w}_base
  CLB_LIB_VARIANT=yinl3 b $w ${w}_yinl3
done
echo done > $O/DONE
