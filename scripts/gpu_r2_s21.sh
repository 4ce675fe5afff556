#!/bin/bash
# round 2 session 21: zero-copy forward_host, copy-out removed; full GPU suite + bench
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s21
timeout 200 python scripts/e2e_probe.py 1 > $O.e2e.log 2>&1
DRK_HOST_OUT=copy timeout 200 python scripts/e2e_probe.py 1 >> $O.e2e.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
