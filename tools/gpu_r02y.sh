#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or cfg3 or step_equals or sharding or odd or simt_repeated" > gpurun_out/y_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/y_pytest_quick.txt
for c in cfg1 cfg2_L14 cfg3; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/y_bench_$c.json 2>> gpurun_out/y_bench.err
  FW_LAT_GENERIC=1 timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/y_bench_${c}_generic.json 2>> gpurun_out/y_bench.err
done
timeout 120 python tools/trace_lat.py cfg1 16 > gpurun_out/y_trace_cfg1.txt 2>&1
