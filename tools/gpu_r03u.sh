#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/fold_check.py 512 40 1 FW_CHAIN_2SM > gpurun_out/u_2sm_512.txt 2>&1; echo "rc=$?" >> gpurun_out/u_2sm_512.txt
timeout 200 python tools/fold_check.py 4096 40 1 FW_CHAIN_2SM > gpurun_out/u_2sm_4096.txt 2>&1; echo "rc=$?" >> gpurun_out/u_2sm_4096.txt
FW_CHAIN_2SM=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/u_bench_2sm.json 2> gpurun_out/u_bench_2sm.err
