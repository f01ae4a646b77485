#!/bin/bash
set -u
O=gpurun_out/r2q; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "pair or x-pair or c4" > $O/pytest_pair.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pair.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 c4lake sw8192 sw8192f32 c2; do
  CLB_CONTIG=pair b $w ${w}_pair
  b $w ${w}_base
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_pair" -s 3 -c 1 \
  -o $O/prof_c4pair env CLB_CONTIG=pair python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $O/ncu_c4pair.log 2>&1
echo done > $O/DONE
