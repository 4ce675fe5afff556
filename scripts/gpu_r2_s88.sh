#!/bin/bash
# round 2 session 88: backward staged batch size (128 = one per thread vs 64 vs 32)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s88
for v in "" vbuild/bb64.so vbuild/bb32.so "" vbuild/bb64.so vbuild/bb32.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; else timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; fi
done > $O.variants.log 2>&1
for v in vbuild/bb64.so vbuild/bb32.so; do
  DRK_LIB_PATH=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_det.py tests/test_gpu_scale.py::test_config2_full_frame_forward_backward -m gpu -q -x > $O.parity_$(basename $v .so).log 2>&1
  echo "rc=$?" >> $O.parity_$(basename $v .so).log
done
