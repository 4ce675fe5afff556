#!/bin/bash
# round 2 session 13: scan-based tie ranking with listed long runs; det trace
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s13
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_det.py -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
DRK_HOST_TRACE=1 DET=1 timeout 400 python scripts/quick_timing.py 1 2 3 > $O.timing.log 2> $O.timing.err
python scripts/one_frame.py 4 > $O.plain_c4.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2s13_launches_c4.csv python scripts/one_frame.py 4 > $O.ncu_c4.log 2>&1
