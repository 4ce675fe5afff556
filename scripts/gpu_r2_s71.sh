#!/bin/bash
# round 2 session 71 (re-entry): restored state — GPU suite, smoke, bench line, quick timing of configs 1-3
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s71
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1
echo "smoke rc=$?" >> $O.smoke.log
timeout 600 python scripts/quick_timing.py 1 2 > $O.quick.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
