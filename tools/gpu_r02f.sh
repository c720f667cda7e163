#!/bin/bash
mkdir -p gpurun_out
python tools/trace_lat.py cfg1 8 > gpurun_out/f_trace_cfg1_c8.txt 2>&1
python tools/trace_lat.py cfg2_L14 16 > gpurun_out/f_trace_cfg2_c16.txt 2>&1
