#!/bin/bash
# round 2 session 62: drk_forward_host pipeline (chunked upload overlapping activation + K1)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s62
timeout 300 python -m pytest tests/test_gpu_fast.py -m gpu -q -x -k "host" > $O.host_tests.log 2>&1
echo "rc=$?" >> $O.host_tests.log
grep -q "rc=0" $O.host_tests.log || exit 0
for i in 1 2; do
timeout 200 python scripts/e2e_probe.py 1 >> $O.e2e.log 2>&1
DRK_H2D_CHUNKS=1 timeout 200 python scripts/e2e_probe.py 1 >> $O.e2e.log 2>&1
done
DRK_H2D_CHUNKS=8 timeout 200 python scripts/e2e_probe.py 1 >> $O.e2e.log 2>&1
DRK_H2D_CHUNKS=2 timeout 200 python scripts/e2e_probe.py 1 >> $O.e2e.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
