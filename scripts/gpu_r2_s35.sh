#!/bin/bash
# round 2 session 35: backward fp64 pass of flagged pixels launched first, beside the fast backward
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s35
for i in 1 2; do
DRK_BWD_CONCURRENT=0 timeout 300 python scripts/quick_timing.py 2 > $O.t0_$i.log 2>&1
timeout 300 python scripts/quick_timing.py 2 > $O.t1_$i.log 2>&1
done
timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
