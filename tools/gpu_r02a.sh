#!/bin/bash
# round-2 GPU session A: tests, FP32 peak, cfg4 bench, per-GPU batch sweep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
./tools/fp32_peak > gpurun_out/a_fp32_peak.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/a_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/a_bench_cfg4.json 2> gpurun_out/a_bench_cfg4.err
for b in 512 1024 2048; do
  timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/a_bench_cfg4_b$b.json 2>> gpurun_out/a_bench_sweep.err
done
