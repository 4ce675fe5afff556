#!/bin/bash
# round 2 session 82c: SH-gradient group sums on the tensor cores, four accumulator chains, padded basis rows (no bank conflicts)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s82c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py::test_config2_full_frame_forward_backward tests/test_golden.py tests/test_gpu_fast.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
for v in "" vbuild/bwd_nomma.so "" vbuild/bwd_nomma.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; else timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; fi
done > $O.variants.log 2>&1
