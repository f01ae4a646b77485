#!/bin/bash
# final bench lines of the committed tree (default line with the CPU leg, reference arm)
set -u
O=gpurun_out/r2z; mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
echo done > $O/DONE
