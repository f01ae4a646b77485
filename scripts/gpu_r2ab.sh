#!/bin/bash
# full -m gpu suite on the committed tree
set -u
O=gpurun_out/r2ab; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
echo done > $O/DONE
