# ncu --set full of the fast raster kernel (config 1) with source correlation; CSV of the source page
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_raster_fast -c 1 -o gpurun_out/ncu_raster_c1 python scripts/one_frame.py 1 > gpurun_out/ncu_raster.log 2>&1
ncu -i gpurun_out/ncu_raster_c1.ncu-rep --page source --csv --print-source cuda > gpurun_out/raster_src.csv 2>/dev/null
ls -la gpurun_out | head
