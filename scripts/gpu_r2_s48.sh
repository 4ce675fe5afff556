#!/bin/bash
# round 2 session 48: onesweep-structured radix sort (one histogram read, one kernel per pass)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s48
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
timeout 400 python scripts/quick_timing.py 1 3 > $O.t1.log 2>&1
DRK_SORT=legacy timeout 400 python scripts/quick_timing.py 1 3 > $O.t0.log 2>&1
timeout 600 python scripts/config4_probe.py 2 > $O.c4_1.log 2>&1
DRK_SORT=legacy timeout 600 python scripts/config4_probe.py 2 > $O.c4_0.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
