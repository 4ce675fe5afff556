#!/bin/bash
# round 2 session 17: concurrent fp64 pass (forward polling consumer, backward beside the fast kernel)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s17
for v in 0 1; do
  DRK_FP64_CONCURRENT=$v timeout 400 python scripts/quick_timing.py 1 2 3 > $O.timing$v.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
