#!/bin/bash
# round 2 session 14: deterministic backward with coalesced row writes and batched reduction
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s14
timeout 900 python -m pytest tests/test_gpu_det.py tests/test_dropin.py tests/test_distributed.py "tests/test_gpu_scale.py::test_config2_full_frame_forward_backward" -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
DRK_HOST_TRACE=1 DET=1 timeout 400 python scripts/quick_timing.py 2 > $O.timing.log 2> $O.timing.err
