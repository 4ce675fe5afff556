#!/bin/bash
# round 2 session 65: radix histogram with per-warp sub-histograms
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s65
for i in 1 2; do timeout 300 python scripts/quick_timing.py 1 3 > $O.t_$i.log 2>&1; done
timeout 900 bash scripts/launch_list.sh 3 $O.launches_c3.csv > $O.launches_c3.md 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > $O.tests.log 2>&1
