#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/trace_fold.py --batch 4096 > gpurun_out/c_trace_4096.txt 2>&1
timeout 120 python tools/trace_fold.py --batch 512 > gpurun_out/c_trace_512.txt 2>&1
