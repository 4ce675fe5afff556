#!/bin/bash
# round 2 session 6: cache-vs-exact probe (current lib + round-1 adapter binary),
# errors tests, early-load variant, config-4 probe after the tie-stat fix
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s6
timeout 300 python scripts/cache_exact_probe.py > $O.probe.log 2>&1
timeout 300 vbuild/r1/a/b/adapter_tests -ts=raster > $O.r1_raster.log 2>&1
DRK_ADAPTER_PRECISION=reference timeout 300 oracle/_ref/adapter_tests -ts=raster > $O.raster_ref.log 2>&1
timeout 600 python -m pytest tests/test_gpu_errors.py tests/test_gpu_fast.py -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
for v in "" vbuild/early.so; do
  echo "== variant: ${v:-product}" >> $O.variants.log
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; else timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; fi
done
timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4probe.log 2>&1
