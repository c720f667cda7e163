#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/t_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/t_pytest.txt
for b in 512 1024 2048 3072; do timeout 120 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/t_bench_b$b.json 2>> gpurun_out/t_bench.err; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/t_bench_cfg4.json 2>> gpurun_out/t_bench.err
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/t_bench_cfg4_200.json 2>> gpurun_out/t_bench.err
FW_CHAIN_SPLIT=1 timeout 400 python tools/race_tc.py 512 600 6 > gpurun_out/t_race_512.txt 2>&1
timeout 400 python tools/race_tc.py 2048 600 4 > gpurun_out/t_race_2048.txt 2>&1
timeout 400 python tools/race_tc.py 384 600 6 > gpurun_out/t_race_384.txt 2>&1
