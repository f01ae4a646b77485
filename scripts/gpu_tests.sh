#!/bin/bash
# GPU tests without -x: TAG "pytest -k expression"
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "$2" -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
echo done > $O/DONE
