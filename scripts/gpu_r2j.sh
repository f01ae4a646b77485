#!/bin/bash
set -u
O=gpurun_out/r2j; mkdir -p $O
CLB_LIB_VARIANT=yinl3 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or slow_path or segmentation or hump or c2_ or slab" > $O/pytest_yinl3.log 2>&1; echo "pytest rc=$?" >> $O/pytest_yinl3.log
CLB_LIB_VARIANT=x32 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or segmentation or slow_path or c5 or sw2048 or c4" > $O/pytest_x32.log 2>&1; echo "pytest rc=$?" >> $O/pytest_x32.log
for w in c4 sw8192 sw8192hump c2 c5 sw8192f32; do
  for v in base yinl3; do
    vv=$v; [ "$v" = base ] && vv=""
    CLB_LIB_VARIANT=$vv timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_${v}.json 2> $O/bench_${w}_${v}.err
  done
done
for w in c4 sw8192 sw8192hump sw8192f32; do
  CLB_LIB_VARIANT=x32 timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_x32.json 2> $O/bench_${w}_x32.err
done
for w in c5 c5f32 c3; do
  CLB_LIB_VARIANT=x32 CLB_CONTIG=tma timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_x32tma.json 2> $O/bench_${w}_x32tma.err
done
echo done > $O/DONE
