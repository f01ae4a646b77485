#!/bin/bash
set -u
O=gpurun_out/r2t; mkdir -p $O
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
CLB_CONTIG=tma b c2 c2_tma
b c2 c2_base
CLB_CONTIG=tma b c1 c1_tma
b c1 c1_base
echo done > $O/DONE
