#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/fold_check.py 512 40 1 FW_CHAIN_2SM 2 > gpurun_out/z_2sf_512.txt 2>&1; echo "rc=$?" >> gpurun_out/z_2sf_512.txt
timeout 200 python tools/fold_check.py 4096 40 1 FW_CHAIN_2SM 2 > gpurun_out/z_2sf_4096.txt 2>&1; echo "rc=$?" >> gpurun_out/z_2sf_4096.txt
FW_CHAIN_2SM=2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/z_bench_2sf.json 2> gpurun_out/z_bench_2sf.err
