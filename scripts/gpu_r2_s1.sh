#!/bin/bash
# round 2, session 1: new GPU tests (deterministic backward, adapter in both
# precisions, acceptance, BASELINE-scale parity), the whole GPU suite, a bench run.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=40 -p no:randomly > gpurun_out/r2s1_gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/r2s1_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2s1_bench.json 2> gpurun_out/r2s1_bench.err
echo "bench rc=$?" >> gpurun_out/r2s1_bench.err
