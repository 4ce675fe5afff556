#!/bin/bash
# round 2 session 2: fixes (fp64 det chain, adapter scratch/fingerprint, banded
# tile lists, C3 view choice) + backward variant timing
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s2
timeout 900 python -m pytest tests/test_gpu_det.py tests/test_dropin.py tests/test_gpu_scale.py -q --durations=30 > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
( time DRK_ADAPTER_TRACE=1 timeout 300 oracle/_ref/adapter_tests -ts=optimize "-tc=single-primitive solid-color smoke fit" ) > $O.trace.log 2>&1
for v in "" vbuild/bwd_smem0.so vbuild/bwd_minb2.so; do
  echo "== variant: ${v:-product}" >> $O.variants.log
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py 2 >> $O.variants.log 2>&1; else timeout 300 python scripts/quick_timing.py 2 >> $O.variants.log 2>&1; fi
done
