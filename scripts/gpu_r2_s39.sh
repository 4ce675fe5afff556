#!/bin/bash
# round 2 session 39: fast backward with one pop_step call site (drain folded into the last batch)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s39
for i in 1 2; do timeout 400 python scripts/quick_timing.py 2 > $O.t_$i.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
