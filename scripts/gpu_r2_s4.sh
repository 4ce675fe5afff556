#!/bin/bash
# round 2 session 4: fp64 SH colours (C4), drop-in + acceptance, full GPU suite
# timing, then ncu (source view) of the fast backward (config 2) and forward (config 1)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s4
DRK_ADAPTER_PRECISION=reference timeout 300 oracle/_ref/fd_probe_adapter > $O.fd_adapter_ref.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
python scripts/one_frame.py 2 bwd > $O.plain_bwd.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd_fast -c 1 \
    -o gpurun_out/r2s4_ncu_bwd python scripts/one_frame.py 2 bwd > $O.ncu_bwd.log 2>&1
python scripts/one_frame.py 1 > $O.plain_fwd.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raster_fast -c 1 \
    -o gpurun_out/r2s4_ncu_fwd python scripts/one_frame.py 1 > $O.ncu_fwd.log 2>&1
ls -la gpurun_out >> $O.ncu_fwd.log
