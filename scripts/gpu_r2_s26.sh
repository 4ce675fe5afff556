#!/bin/bash
# round 2 session 26: fp64 per-pixel kernels, compositing from per-warp shared slots
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s26
timeout 400 python scripts/quick_timing.py 1 2 3 > $O.timing.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 600 python scripts/config4_probe.py 1 bwd > $O.c4probe.log 2>&1
