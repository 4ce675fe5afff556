#!/bin/bash
# round 2 session 15: two-level deterministic reduction; band-cache margin; config-4 probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s15
timeout 900 python -m pytest tests/test_gpu_det.py tests/test_dropin.py "tests/test_gpu_scale.py::test_config2_full_frame_forward_backward" "tests/test_gpu_scale.py::test_config4_band" -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
DRK_HOST_TRACE=1 DET=1 timeout 400 python scripts/quick_timing.py 2 > $O.timing.log 2> $O.timing.err
timeout 900 python scripts/config4_probe.py 3 bwd > $O.c4probe.log 2>&1
