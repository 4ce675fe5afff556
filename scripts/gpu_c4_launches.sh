# per-kernel launch list of one config-4 forward (4M DRK, 3840x2160, banded)
timeout 1500 bash scripts/launch_list.sh 4 gpurun_out/launches_c4.csv > gpurun_out/launches_c4.md 2>&1
cat gpurun_out/launches_c4.md
