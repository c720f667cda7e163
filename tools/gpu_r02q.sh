#!/bin/bash
mkdir -p gpurun_out
for k in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 300 -k split > gpurun_out/q_pytest_split_$k.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest_split_$k.txt
done
for b in 512 2048; do timeout 120 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/q_bench_b$b.json 2>> gpurun_out/q_bench.err; done
