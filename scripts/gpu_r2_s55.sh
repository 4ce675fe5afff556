#!/bin/bash
# round 2 session 55: SortCache pop-through fast path in the fast forward
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s55
for v in base thru_stat thru; do
  if [ $v = base ]; then L=""; else L=vbuild/$v.so; fi
  DRK_LIB_PATH=$L timeout 300 python scripts/quick_timing.py 1 2 3 > $O.$v.log 2>&1
done
DRK_LIB_PATH=vbuild/thru.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fast.py -m gpu -q -x > $O.tests.log 2>&1
