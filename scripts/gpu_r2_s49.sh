#!/bin/bash
# round 2 session 49: onesweep-structured radix sort, tile counters zeroed
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s49
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
grep -q "rc=0" $O.parity.log || exit 0
timeout 300 python scripts/quick_timing.py 1 3 > $O.t1.log 2>&1
DRK_SORT=legacy timeout 300 python scripts/quick_timing.py 1 3 > $O.t0.log 2>&1
timeout 400 python scripts/config4_probe.py 2 > $O.c4_1.log 2>&1
DRK_SORT=legacy timeout 400 python scripts/config4_probe.py 2 > $O.c4_0.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
