#!/bin/bash
# round-2 GPU session C: the small-batch cluster kernel (cell_lat.cu), prefill GEMMs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cluster or cfg1 or small_batch or cfg2 or prefill or naive or step_equals or sharding or odd" > gpurun_out/c_pytest_quick.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c_pytest_quick.txt
timeout 600 python bench.py --config cfg1 --steps 500 --warmup 10 --cpu-seconds 5 > gpurun_out/c_bench_cfg1.json 2> gpurun_out/c_bench_cfg1.err
for c in 8 16; do FW_SIMT_CLUSTER=$c timeout 300 python bench.py --config cfg2_L14 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/c_bench_cfg2_L14_c$c.json 2>> gpurun_out/c_bench_cfg2.err; done
FW_SIMT_CLUSTER=16 timeout 300 python bench.py --config cfg1 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/c_bench_cfg1_c16.json 2>> gpurun_out/c_bench_cfg1.err
timeout 600 python tools/depth_sweep.py --steps 1000 --naive-steps 20 > gpurun_out/c_depth_sweep.jsonl 2> gpurun_out/c_depth_sweep.err
timeout 300 python tools/profile_prefill.py cfg5 64 > gpurun_out/c_prefill_cfg5.txt 2>&1
timeout 300 python tools/profile_prefill.py cfg3 500 >> gpurun_out/c_prefill_cfg5.txt 2>&1
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/c_lat_cfg1 python tools/profile_step.py 50 cfg1 > gpurun_out/c_ncu_lat.log 2>&1
timeout 1200 ncu --replay-mode app-range --profile-from-start off --set full --clock-control none -o gpurun_out/c_step_range python tools/profile_step.py 10 cfg4 > gpurun_out/c_ncu_range.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/c_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c_pytest.txt
