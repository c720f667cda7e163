#!/bin/bash
# session r03b: first run of the folded chain
mkdir -p gpurun_out
timeout 120 python tools/fold_check.py 512 40 > gpurun_out/b_fold_512.txt 2>&1; echo "rc=$?" >> gpurun_out/b_fold_512.txt
timeout 200 python tools/fold_check.py 4096 40 > gpurun_out/b_fold_4096.txt 2>&1; echo "rc=$?" >> gpurun_out/b_fold_4096.txt
timeout 300 python tools/fold_check.py 4096 600 3 > gpurun_out/b_fold_4096_600.txt 2>&1; echo "rc=$?" >> gpurun_out/b_fold_4096_600.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_bench_fold.json 2> gpurun_out/b_bench_fold.err
FW_CHAIN_FOLD=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_bench_nofold.json 2> gpurun_out/b_bench_nofold.err
timeout 300 python bench.py --steps 50 --warmup 5 --batch 512 --no-cpu-baseline > gpurun_out/b_bench_fold_512.json 2>> gpurun_out/b_bench_fold.err
