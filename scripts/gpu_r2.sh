#!/bin/bash
# Round-2 GPU session: host facts, smoke, the full -m gpu suite (with the new
# BASELINE-size and per-variant parity tests), the default bench line (C4)
# and the reference arm.  Usage: gpurun --timeout 2400 -- 'bash scripts/gpu_r2.sh TAG'
set -u
TAG=${1:-r2}
O=gpurun_out/$TAG
mkdir -p $O
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv; } > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
echo done > $O/DONE
