#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/trace_fold.py --batch 4096 > gpurun_out/d_trace_4096.txt 2>&1
timeout 200 python tools/fold_check.py 4096 600 2 > gpurun_out/d_fold_4096_600.txt 2>&1; echo "rc=$?" >> gpurun_out/d_fold_4096_600.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/d_bench_fold.json 2> gpurun_out/d_bench_fold.err
timeout 300 python bench.py --steps 50 --warmup 5 --batch 512 --no-cpu-baseline > gpurun_out/d_bench_fold_512.json 2>> gpurun_out/d_bench_fold.err
