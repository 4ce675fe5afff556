#!/bin/bash
# round 2 session 38: ncu source view of the current fast backward (config 2, half-tile CTAs)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s38
python scripts/one_frame.py 2 bwd > $O.plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd_fast -c 1 \
    -o gpurun_out/r2s38_ncu_bwd python scripts/one_frame.py 2 bwd > $O.ncu.log 2>&1
echo "rc=$?" >> $O.ncu.log
