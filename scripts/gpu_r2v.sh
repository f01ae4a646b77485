#!/bin/bash
set -u
O=gpurun_out/r2v; mkdir -p $O
CLB_LIB_VARIANT=r96m4 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or sw2048 or segmentation or c5" > $O/pytest_r96m4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_r96m4.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 sw8192 sw8192hump sw8192f32 c5 c5f32; do
  CLB_LIB_VARIANT=r96m4 b $w ${w}_r96m4
done
echo done > $O/DONE
