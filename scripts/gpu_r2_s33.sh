#!/bin/bash
# round 2 session 33: K1 bitonic sort, 2 (default) / 3 stages per shared-memory round trip
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s33
timeout 400 python scripts/quick_timing.py 1 3 > $O.timing.log 2>&1
DRK_LIB_PATH=vbuild/prep_sort3.so timeout 400 python scripts/quick_timing.py 1 3 > $O.timing3.log 2>&1
DRK_LIB_PATH=vbuild/prep_sort3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > $O.tests3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
