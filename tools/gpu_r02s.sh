#!/bin/bash
mkdir -p gpurun_out
FW_CHAIN_SPLIT=0 timeout 400 python tools/race_tc.py 1152 600 8 > gpurun_out/s_race_1152_nosplit.txt 2>&1
FW_CHAIN_SPLIT=1 timeout 400 python tools/race_tc.py 1152 600 8 > gpurun_out/s_race_1152_split.txt 2>&1
timeout 600 python tools/race_tc.py 4096 600 4 > gpurun_out/s_race_4096.txt 2>&1
