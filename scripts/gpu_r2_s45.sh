#!/bin/bash
# round 2 session 45: deterministic backward with half-tile CTAs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s45
DET=1 DRK_HOST_TRACE=1 timeout 400 python scripts/quick_timing.py 2 > $O.t256.log 2>&1
DRK_DET_NT=128 DET=1 DRK_HOST_TRACE=1 timeout 400 python scripts/quick_timing.py 2 > $O.t128.log 2>&1
DRK_DET_NT=128 timeout 900 python -m pytest tests/test_gpu_det.py tests/test_dropin.py -m gpu -q -x > $O.tests128.log 2>&1
