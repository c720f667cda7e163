#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/p_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/p_pytest.txt
for b in 512 1024 2048 3072; do timeout 120 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/p_bench_b$b.json 2>> gpurun_out/p_bench.err; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/p_bench_cfg4.json 2>> gpurun_out/p_bench.err
