#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/h_lat_cfg2 python tools/profile_step.py 20 cfg2_L14 > gpurun_out/h_ncu.log 2>&1
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/h_lat_cfg1 python tools/profile_step.py 50 cfg1 >> gpurun_out/h_ncu.log 2>&1
