#!/bin/bash
# round 2 session 9: parallel tie ordering, cache-append statistic
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s9
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fast.py tests/test_gpu_det.py -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
timeout 300 python scripts/quick_timing.py 1 2 > $O.timing.log 2>&1
timeout 300 python scripts/quick_timing.py 3 >> $O.timing.log 2>&1
timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4probe.log 2>&1
