#!/bin/bash
# round 2 session 81: K1 interior-point filter before the vertex sort — parity at scale, timing A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s81
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_vcache.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
for v in "" vbuild/k1nofilt.so "" vbuild/k1nofilt.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-fwd-bwd --no-config4-train --no-adapter --no-train --no-cpu-baseline > $O.mv.json 2> $O.mv.err
DRK_LIB_PATH=vbuild/k1nofilt.so timeout 600 python bench.py --steps 5 --warmup 3 --no-fwd-bwd --no-config4-train --no-adapter --no-train --no-cpu-baseline > $O.mv_off.json 2> $O.mv_off.err
