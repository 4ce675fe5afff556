#!/bin/bash
# round 2 session 16: full GPU suite + smoke + bench (det budget)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s16
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1
DRK_HOST_TRACE=1 DET=1 timeout 400 python scripts/quick_timing.py 2 > $O.timing.log 2> $O.timing.err
timeout 1500 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
