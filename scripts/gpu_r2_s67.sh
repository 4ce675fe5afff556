#!/bin/bash
# round 2 session 67: config 1 with half-tile CTAs (pop-through compiled in) vs whole tiles
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s67
for i in 1 2; do
timeout 300 python scripts/quick_timing.py 1 > $O.rk0_$i.log 2>&1
RK=6 timeout 300 python scripts/quick_timing.py 1 > $O.rk6_$i.log 2>&1
done
