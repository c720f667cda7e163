#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or step_equals or sharding or odd" > gpurun_out/k_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/k_pytest_quick.txt
for cfg in cfg1 cfg2_L14; do for c in 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config $cfg --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/k_bench_${cfg}_c$c.json 2>> gpurun_out/k_bench.err; done; done
FW_SIMT_CLUSTER=2 timeout 300 python bench.py --config cfg3 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/k_bench_cfg3_c2.json 2>> gpurun_out/k_bench.err
python tools/trace_lat.py cfg3 2 > gpurun_out/k_trace_cfg3_c2.txt 2>&1
python tools/trace_lat.py cfg1 8 > gpurun_out/k_trace_cfg1_c8.txt 2>&1
python tools/trace_lat.py cfg2_L14 16 > gpurun_out/k_trace_cfg2_c16.txt 2>&1
