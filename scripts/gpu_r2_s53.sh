#!/bin/bash
# round 2 session 53: bench under torchrun (world 1) with the light legs, reference arm under torchrun
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s53
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-config4-train --no-adapter --no-cpu-baseline --multiview-views 8 > $O.tr.json 2> $O.tr.err
echo "rc=$?" >> $O.tr.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > $O.ref.json 2> $O.ref.err
echo "rc=$?" >> $O.ref.err
