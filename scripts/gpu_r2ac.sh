#!/bin/bash
# streaming twin at a 3-CTA register target (194 registers, no stack)
set -u
O=gpurun_out/r2ac; mkdir -p $O
CLB_LIB_VARIANT=xs3 timeout 600 python -m pytest tests -m gpu -x -q -k "streaming or geometry_pair" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 sw8192 c4lake; do
  CLB_LIB_VARIANT=xs3 b $w ${w}_xs3
  b $w ${w}_default
done
echo done > $O/DONE
