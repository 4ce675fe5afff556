#!/bin/bash
# round 2 session 34: bench after the key / K1 / fp64-pass changes
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s34
timeout 1200 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1
echo "smoke rc=$?" >> $O.smoke.log
