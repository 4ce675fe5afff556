#!/bin/bash
# round 2 session 23: K1 prep, larger wedge stacks
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s23
for v in prep_w4_s96 prep_w4_s128 prep_w4_s160 prep_w2_s128; do
  DRK_LIB_PATH=vbuild/$v.so timeout 300 python scripts/quick_timing.py 1 3 > $O.$v.log 2>&1
done
