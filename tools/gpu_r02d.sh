#!/bin/bash
# round-2 GPU session D: the small-batch kernel with st.async exchanges
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or cfg3 or prefill or naive or step_equals or sharding or odd or staged" > gpurun_out/d_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/d_pytest_quick.txt
for c in 2 4 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg1 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/d_bench_cfg1_c$c.json 2>> gpurun_out/d_bench.err; done
for c in 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg2_L14 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/d_bench_cfg2_L14_c$c.json 2>> gpurun_out/d_bench.err; done
for c in 0 2; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg3 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/d_bench_cfg3_c$c.json 2>> gpurun_out/d_bench.err; done
timeout 600 python tools/depth_sweep.py --steps 1000 --naive-steps 20 > gpurun_out/d_depth_sweep.jsonl 2> gpurun_out/d_depth_sweep.err
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/d_lat_cfg1 python tools/profile_step.py 50 cfg1 > gpurun_out/d_ncu_lat.log 2>&1
