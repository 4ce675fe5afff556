#!/bin/bash
# round 2 session 41: reference-precision forward / backward as thread-per-pixel kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s41
timeout 300 python scripts/fp64_all_probe.py > $O.probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O.bench.json 2> $O.bench.err
