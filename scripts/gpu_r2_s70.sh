#!/bin/bash
# round 2 session 70: K1 vertex cache (multi-view)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s70
timeout 300 python -m pytest tests/test_gpu_vcache.py -m gpu -q -x > $O.vc_test.log 2>&1
echo "rc=$?" >> $O.vc_test.log
grep -q "rc=0" $O.vc_test.log || exit 0
A="--steps 3 --warmup 3 --no-fwd-bwd --no-config4-train --no-adapter --no-train --no-cpu-baseline"
timeout 900 python bench.py $A > $O.on.json 2> $O.on.err
DRK_VCACHE=0 timeout 900 python bench.py $A > $O.off.json 2> $O.off.err
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
