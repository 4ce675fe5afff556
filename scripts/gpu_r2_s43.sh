#!/bin/bash
# round 2 session 44: adapter staging in page-locked grow-only buffers
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s43
timeout 600 python scripts/adapter_trace.py fast > $O.fast.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
