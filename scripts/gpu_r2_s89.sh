#!/bin/bash
# round 2 session 89: final checkpoint after the backward batch-size change — GPU suite, smoke, bench, reference arm, launch list, ncu of the forward raster
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s89
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1
echo "smoke rc=$?" >> $O.smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O.bench_ref.json 2> $O.bench_ref.err
timeout 900 bash scripts/launch_list.sh 1 $O.launches_c1.csv > $O.launches_c1.md 2>&1
python scripts/one_frame.py 1 > $O.plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raster_fast -c 1 \
    -o gpurun_out/r2s89_ncu_fwd python scripts/one_frame.py 1 > $O.ncu.log 2>&1
echo "ncu rc=$?" >> $O.ncu.log
