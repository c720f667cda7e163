#!/bin/bash
mkdir -p gpurun_out
timeout 500 python tools/race_split2.py 512 4 > gpurun_out/r_race2_512.txt 2>&1
timeout 500 python tools/race_split2.py 1152 3 > gpurun_out/r_race2_1152.txt 2>&1
