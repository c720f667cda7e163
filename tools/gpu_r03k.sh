#!/bin/bash
mkdir -p gpurun_out
for k in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider -k "tcgen05_repeated" > gpurun_out/k_race_$k.txt 2>&1; echo "rc=$?" >> gpurun_out/k_race_$k.txt
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "warp_mma or cfg5 or simt_repeated or staged" > gpurun_out/k_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.txt
timeout 300 python bench.py --config cfg5 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/k_bench_cfg5.json 2>/dev/null
timeout 120 python tools/trace_hmma.py cfg5 > gpurun_out/k_trace.txt 2>&1
