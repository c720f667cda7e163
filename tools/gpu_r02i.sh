#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/i_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/i_pytest.txt
for c in 0 2 4; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg3 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/i_bench_cfg3_c$c.json 2>> gpurun_out/i_bench.err; done
timeout 600 python tools/depth_sweep.py --steps 1000 --naive-steps 20 > gpurun_out/i_depth_sweep.jsonl 2> gpurun_out/i_depth_sweep.err
python tools/trace_lat.py cfg3 2 > gpurun_out/i_trace_cfg3_c2.txt 2>&1
