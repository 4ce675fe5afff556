#!/bin/bash
# round 2 session 37: backward tiles dispatched by the forward's streamed length
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s37
for i in 1 2; do
DRK_BWD_ORDER=0 timeout 400 python scripts/quick_timing.py 2 > $O.t0_$i.log 2>&1
timeout 400 python scripts/quick_timing.py 2 > $O.t1_$i.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
