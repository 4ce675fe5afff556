#!/bin/bash
# round 2 session 60: GPU suite with the backward pop-through path on
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s60
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 300 python scripts/quick_timing.py 2 > $O.t.log 2>&1
