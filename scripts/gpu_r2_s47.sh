#!/bin/bash
# round 2 session 47: one barrier less per batch in both raster kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s47
for i in 1 2; do timeout 400 python scripts/quick_timing.py 1 2 > $O.t_$i.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
