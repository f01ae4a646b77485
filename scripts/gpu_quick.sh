#!/bin/bash
# Quick GPU iteration: gpu tests (optional), a few bench lines, optional ncu capture.
# Usage: gpurun -- 'bash scripts/gpu_quick.sh TAG "c2 sw8192" [tests] [ncu:WORKLOAD]'
set -u
TAG=$1; WL=${2:-"sw8192"}; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for x in "$@"; do
  case $x in
    tests) timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log;;
    tests:*) timeout 900 python -m pytest tests -m gpu -x -q -k "${x#tests:}" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log;;
  esac
done
# a workload "name@variant" runs with CLB_LIB_VARIANT=variant (libclawb200_<variant>.so)
for w in $WL; do
  name=${w%@*}; var=""; [ "$name" != "$w" ] && var=${w#*@}
  CLB_LIB_VARIANT=$var timeout 400 python bench.py --workload $name --steps 20 --warmup 5 --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
for x in "$@"; do
  case $x in
    ncu:*) w=${x#ncu:}; name=${w%@*}; var=""; [ "$name" != "$w" ] && var=${w#*@}
      CLB_LIB_VARIANT=$var timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 6 -c 2 \
        -o $O/prof_$w python bench.py --workload $name --steps 2 --warmup 3 --no-cpu > $O/ncu_$w.log 2>&1;;
    py:*) timeout 600 python ${x#py:} > $O/$(basename ${x#py:}).log 2>&1;;
  esac
done
echo done > $O/DONE
