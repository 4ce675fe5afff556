#!/bin/bash
# round 2 session 19: zero-copy host-buffer forward (mapped outputs / inputs)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s19
for c in 1 2; do
  DRK_HOST_OUT=copy timeout 300 python scripts/e2e_probe.py $c >> $O.e2e.log 2>&1
  timeout 300 python scripts/e2e_probe.py $c >> $O.e2e.log 2>&1
  DRK_HOST_IN=map timeout 300 python scripts/e2e_probe.py $c >> $O.e2e.log 2>&1
  DRK_HOST_OUT=copy DRK_HOST_IN=map timeout 300 python scripts/e2e_probe.py $c >> $O.e2e.log 2>&1
done
timeout 600 python -m pytest tests -m gpu -q -x -k "host or e2e or forward_host or smoke" > $O.tests.log 2>&1
