#!/bin/bash
# round 2 session 3: C4 probe, adapter replay speed, comm, distributed, TMA/ISECT2 A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s3
DRK_ADAPTER_PRECISION=reference timeout 300 oracle/_ref/fd_probe_adapter > $O.fd_adapter_ref.txt 2>&1
DRK_ADAPTER_PRECISION=fast timeout 300 oracle/_ref/fd_probe_adapter > $O.fd_adapter_fast.txt 2>&1
( time DRK_ADAPTER_TRACE=1 timeout 300 oracle/_ref/adapter_tests -ts=optimize "-tc=single-primitive solid-color smoke fit" ) > $O.trace.log 2>&1
timeout 900 python -m pytest tests/test_comm.py tests/test_distributed.py tests/test_gpu_det.py tests/test_gpu_parity.py tests/test_gpu_fast.py "tests/test_gpu_scale.py::test_config4_band" -q -m gpu --durations=15 > $O.tests.log 2>&1
echo "rc=$?" >> $O.tests.log
for v in "" vbuild/notma.so vbuild/isect2.so; do
  echo "== variant: ${v:-product}" >> $O.variants.log
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; else timeout 300 python scripts/quick_timing.py 1 2 >> $O.variants.log 2>&1; fi
done
