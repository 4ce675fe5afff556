#!/bin/bash
# round 2 session 77: early-bracket product (default on) vs next-entry prefetch
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s77
for v in "" vbuild/pfn.so "" vbuild/pfn.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
