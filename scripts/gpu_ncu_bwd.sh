# ncu --set full of the fast backward rasterizer (config 2) and of one radix scatter pass (config 3 scale)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd_fast -c 1 -o gpurun_out/ncu_bwd_fast python scripts/one_frame.py 2 bwd > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rs_scatter -c 1 -o gpurun_out/ncu_scatter_c3 python scripts/one_frame.py 3 > gpurun_out/ncu_scatter.log 2>&1
ls -la gpurun_out
