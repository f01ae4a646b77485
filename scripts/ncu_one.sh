#!/bin/bash
# ncu --set full of the sweep kernels of one workload: TAG WORKLOAD [ENV=VAL ...]
O=gpurun_out/$1; W=$2; shift 2; mkdir -p $O
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 6 -c 1 \
  -o $O/prof_${W}$(printf '_%s' "$@" | tr '=' '-') python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $O/ncu_$W.log 2>&1
