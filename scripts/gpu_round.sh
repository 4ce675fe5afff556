set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python scripts/quick_timing.py 0 1 2 > gpurun_out/quick.log 2>&1
timeout 600 bash scripts/launch_list.sh 1 gpurun_out/launches_c1.csv > gpurun_out/launches_c1.md 2>&1
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench.json; cat gpurun_out/quick.log | cut -c1-400
