#!/bin/bash
# round 2 session 86: shape-record lookup angles staged in the ring record (forward + backward / forward only / off)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s86
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fast.py tests/test_gpu_scale.py::test_config1_full_frame -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
for v in "" vbuild/rs_bwdoff.so vbuild/rs_off.so "" vbuild/rs_bwdoff.so vbuild/rs_off.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-420; else timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-420; fi
done > $O.variants.log 2>&1
