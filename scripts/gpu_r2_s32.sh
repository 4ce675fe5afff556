#!/bin/bash
# round 2 session 32: NearestDepth keys with one division (emit + tie keys)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s32
timeout 400 python scripts/quick_timing.py 1 3 > $O.timing.log 2>&1
timeout 600 python scripts/config4_probe.py 2 > $O.c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
