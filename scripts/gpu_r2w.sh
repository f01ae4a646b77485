#!/bin/bash
# x geometry pair (CLB_XVAR_TMA_ADAPT): parity of the streaming twin and the
# paired launch, then A/B against each geometry alone
set -u
O=gpurun_out/r2w; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "streaming or golden_sweeps or sw2048 or segmentation or slow_path or c4 or hump or sw8192 or golden_runs" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 sw8192 sw8192hump; do
  b $w ${w}_adapt
  CLB_CONTIG=tma b $w ${w}_tma
  CLB_CONTIG=stream b $w ${w}_stream
done
b c4lake c4lake_adapt
CLB_XS_FRAC=0.02 b c4 c4_frac02
CLB_XS_FRAC=0.3 b sw8192 sw8192_frac30
echo done > $O/DONE
