#!/bin/bash
# round 2 session 42: adapter phase trace (config 2)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s42
timeout 600 python scripts/adapter_trace.py fast > $O.fast.log 2>&1
timeout 600 python scripts/adapter_trace.py reference > $O.ref.log 2>&1
