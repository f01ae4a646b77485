#!/bin/bash
# One GPU session: parity tests, bench lines, ncu launch list + full capture.
# Usage (from this container):  gpurun --timeout 1500 -- 'bash scripts/gpu_session.sh [tag]'
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in c2 sw8192 sw8192hump sw8192f32 c1 c3 c4 c5 c5f32; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 $( [ $w != c2 ] && echo --no-cpu ) > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
# launch list (cold-cache, serialised): shares only
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/launches_c2.csv python bench.py --workload c2 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file $O/launches_sw8192.csv python bench.py --workload sw8192 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
# full capture of the two sweep kernels on the north-star grid
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|sweep_contig" -s 6 -c 2 \
  -o $O/prof_sw8192 python bench.py --workload sw8192 --steps 3 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|sweep_contig" -s 6 -c 2 \
  -o $O/prof_c2 python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu > $O/ncu_full_c2.log 2>&1
echo done > $O/DONE
