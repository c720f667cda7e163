#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/trace_hmma.py cfg5 > gpurun_out/g_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 600 -k "cfg5 or cfg3" -rf > gpurun_out/g_pytest_long.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/g_pytest_long.txt
for c in cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/g_bench_$c.json 2>> gpurun_out/g_bench.err
done
FW_HMMA_NT=2 timeout 300 python bench.py --config cfg5 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/g_bench_cfg5_nt2.json 2>> gpurun_out/g_bench.err
