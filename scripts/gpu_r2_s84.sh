#!/bin/bash
# round 2 session 84: 128-entry batches in the whole-tile forward (half the ring / staging shared memory)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s84
for v in "" vbuild/b128.so "" vbuild/b128.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
DRK_LIB_PATH=vbuild/b128.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fast.py tests/test_gpu_scale.py::test_config1_full_frame -m gpu -q -x > $O.parity_b128.log 2>&1
echo "rc=$?" >> $O.parity_b128.log
