#!/bin/bash
# round 2 session 25: ncu source view of the fp64 per-pixel kernels (config 2, forward + backward)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s25
python scripts/one_frame.py 2 bwd > $O.plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raster_pixels_warp -c 2 \
    -o gpurun_out/r2s25_ncu_warp python scripts/one_frame.py 2 bwd > $O.ncu.log 2>&1
echo "rc=$?" >> $O.ncu.log
