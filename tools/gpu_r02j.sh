#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or cfg3 or step_equals or sharding or odd or staged" > gpurun_out/j_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/j_pytest_quick.txt
for cfg in cfg1 cfg2_L14; do for c in 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config $cfg --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/j_bench_${cfg}_c$c.json 2>> gpurun_out/j_bench.err; done; done
for c in 2 4; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg3 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/j_bench_cfg3_c$c.json 2>> gpurun_out/j_bench.err; done
python tools/trace_lat.py cfg3 2 > gpurun_out/j_trace_cfg3_c2.txt 2>&1
python tools/trace_lat.py cfg1 16 > gpurun_out/j_trace_cfg1_c16.txt 2>&1
