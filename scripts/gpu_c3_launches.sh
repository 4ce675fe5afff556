timeout 900 bash scripts/launch_list.sh 3 gpurun_out/launches_c3.csv > gpurun_out/launches_c3.md 2>&1
cat gpurun_out/launches_c3.md
