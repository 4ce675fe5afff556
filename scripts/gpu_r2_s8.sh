#!/bin/bash
# round 2 session 8: full GPU suite, smoke, bench, reference arm, launch list (config 1)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s8
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > $O.gpu_tests.log 2>&1
echo "rc=$?" >> $O.gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O.bench.json 2> $O.bench.err
echo "bench rc=$?" >> $O.bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O.bench_ref.json 2> $O.bench_ref.err
python scripts/one_frame.py 1 2 > $O.plain_c1.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2s8_launches_c1.csv python scripts/one_frame.py 1 2 > $O.ncu_launch.log 2>&1
