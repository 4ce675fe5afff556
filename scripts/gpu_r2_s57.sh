#!/bin/bash
# round 2 session 57: pop-through fast path in the half-tile forward kernel only
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s57
timeout 300 python scripts/quick_timing.py 1 2 3 > $O.t.log 2>&1
timeout 400 python scripts/config4_probe.py 2 > $O.c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
