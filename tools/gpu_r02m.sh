#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 600 -x -k split > gpurun_out/m_pytest_split.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/m_pytest_split.txt
for b in 512 1024 2048 3072; do
  timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/m_bench_b$b.json 2>> gpurun_out/m_bench.err
  FW_CHAIN_SPLIT=0 timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/m_bench_b${b}_nosplit.json 2>> gpurun_out/m_bench.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "tcgen05 or cfg4" > gpurun_out/m_pytest_tc.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/m_pytest_tc.txt
