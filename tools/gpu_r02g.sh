#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or step_equals or sharding or odd" > gpurun_out/g_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/g_pytest_quick.txt
python tools/trace_lat.py cfg1 8 > gpurun_out/g_trace_cfg1_c8.txt 2>&1
python tools/trace_lat.py cfg2_L14 16 > gpurun_out/g_trace_cfg2_c16.txt 2>&1
for c in 4 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg1 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/g_bench_cfg1_c$c.json 2>> gpurun_out/g_bench.err; done
for c in 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg2_L14 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/g_bench_cfg2_L14_c$c.json 2>> gpurun_out/g_bench.err; done
