#!/bin/bash
# round 2 session 36: flagged pixels ordered by composite count before the fp64 passes
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s36
for i in 1 2; do
DRK_REDO_ORDER=0 timeout 400 python scripts/quick_timing.py 1 2 3 > $O.t0_$i.log 2>&1
timeout 400 python scripts/quick_timing.py 1 2 3 > $O.t1_$i.log 2>&1
done
DRK_REDO_ORDER=0 timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4_0.log 2>&1
timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4_1.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
