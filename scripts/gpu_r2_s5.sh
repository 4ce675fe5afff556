#!/bin/bash
# round 2 session 5: drop-in fix check, backward CTA-shape variants, config-4 tie stats, bench
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s5
timeout 900 python -m pytest tests/test_dropin.py tests/test_gpu_det.py tests/test_comm.py -q -m gpu > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
for v in "" "NT128" "vbuild/bwd128m3.so"; do
  echo "== variant: ${v:-product}" >> $O.variants.log
  case "$v" in
    "") timeout 300 python scripts/quick_timing.py 2 >> $O.variants.log 2>&1 ;;
    NT128) DRK_BWD_NT=128 timeout 300 python scripts/quick_timing.py 2 >> $O.variants.log 2>&1 ;;
    *) DRK_BWD_NT=128 DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py 2 >> $O.variants.log 2>&1 ;;
  esac
done
timeout 600 python scripts/config4_probe.py 2 bwd > $O.c4probe.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
