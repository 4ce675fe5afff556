#!/bin/bash
# round 2 session 31: K1 vertex sort in registers
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s31
timeout 400 python scripts/quick_timing.py 1 3 > $O.timing.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
