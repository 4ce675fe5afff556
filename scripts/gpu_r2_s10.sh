#!/bin/bash
# round 2 session 10: launch lists of a config-4 view (forward) and a config-3 view
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s10
python scripts/one_frame.py 4 > $O.plain_c4.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2s10_launches_c4.csv python scripts/one_frame.py 4 > $O.ncu_c4.log 2>&1
python scripts/one_frame.py 3 > $O.plain_c3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2s10_launches_c3.csv python scripts/one_frame.py 3 > $O.ncu_c3.log 2>&1
