#!/bin/bash
# round 2 session 30: ncu source view of K1 (k_prep_warp, config 3 view 0)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s30
python scripts/one_frame.py 3 > $O.plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_prep_warp -c 1 \
    -o gpurun_out/r2s30_ncu_prep python scripts/one_frame.py 3 > $O.ncu.log 2>&1
echo "rc=$?" >> $O.ncu.log
