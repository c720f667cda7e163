#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/race_tc.py 2048 600 12 > gpurun_out/v_race_2048.txt 2>&1
FW_CHAIN_SPLIT=0 timeout 900 python tools/race_tc.py 2048 600 6 > gpurun_out/v_race_2048_nosplit.txt 2>&1
timeout 900 python tools/race_tc.py 4096 600 5 > gpurun_out/v_race_4096.txt 2>&1
for b in 512 2048; do timeout 120 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/v_bench_b$b.json 2>> gpurun_out/v_bench.err; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v_bench_cfg4.json 2>> gpurun_out/v_bench.err
