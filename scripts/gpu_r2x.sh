#!/bin/bash
# streaming twin with two 128-B boxes per row and stage (256 B of each row
# per stage): 32 rows x 3 CTAs (s2r32) or 64 rows x 1 CTA (s2r64)
set -u
O=gpurun_out/r2x; mkdir -p $O
for v in s2r32 s2r64 default; do
  if [ $v = default ]; then V=""; else V=$v; fi
  CLB_LIB_VARIANT=$V timeout 900 python -m pytest tests -m gpu -x -q -k "streaming or sw2048 or golden_sweeps" > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
done
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for v in s2r32 s2r64 default; do
  if [ $v = default ]; then V=""; else V=$v; fi
  CLB_LIB_VARIANT=$V CLB_CONTIG=stream b c4lake lake_stream_$v
  CLB_LIB_VARIANT=$V b c4 c4_adapt_$v
  CLB_LIB_VARIANT=$V b sw8192 sw8192_adapt_$v
done
CLB_CONTIG=tma b c4lake lake_tma_default
b sw8192hump hump_adapt_default
echo done > $O/DONE
