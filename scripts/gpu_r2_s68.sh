#!/bin/bash
# round 2 session 68: multiview with 1 / 2 / 3 in-flight contexts
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s68
A="--steps 3 --warmup 3 --no-fwd-bwd --no-config4-train --no-adapter --no-train --no-cpu-baseline"
for f in 1 2 3; do
timeout 900 python bench.py $A --multiview-inflight $f > $O.if$f.json 2> $O.if$f.err
done
