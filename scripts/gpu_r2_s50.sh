#!/bin/bash
# round 2 session 50: onesweep sort launch list (config 1) + ncu of one pass
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s50
timeout 600 bash scripts/launch_list.sh 1 $O.launches_c1.csv > $O.launches_c1.md 2>&1
timeout 600 bash scripts/launch_list.sh 3 $O.launches_c3.csv > $O.launches_c3.md 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_os_pass -s 4 -c 1 \
    -o gpurun_out/r2s50_ncu_os python scripts/one_frame.py 3 > $O.ncu.log 2>&1
