#!/bin/bash
# round 2 session 7: bitwise cache/exact (alpha64), drop-in + acceptance, cache fast-path variants
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s7
timeout 300 python scripts/cache_exact_probe.py > $O.probe.log 2>&1
timeout 900 python -m pytest tests/test_dropin.py -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
for v in "" vbuild/cfast.so vbuild/cfast_early.so; do
  echo "== variant: ${v:-product}" >> $O.variants.log
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; else timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; fi
done
