#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 300 -x -k split > gpurun_out/o_pytest_split.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/o_pytest_split.txt
for b in 512 2048; do timeout 120 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/o_bench_b$b.json 2>> gpurun_out/o_bench.err; done
timeout 120 python tools/trace_chain.py --batch 512 > gpurun_out/o_trace_split.txt 2>&1
