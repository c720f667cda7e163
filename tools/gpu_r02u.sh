#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/race_tc.py 2048 600 12 > gpurun_out/u_race_2048_nofence.txt 2>&1
cp paper_1611_09482_b200/libfastwavenet.so /tmp/nofence.so
cp paper_1611_09482_b200/libfastwavenet_fence.so paper_1611_09482_b200/libfastwavenet.so
timeout 900 python tools/race_tc.py 2048 600 12 > gpurun_out/u_race_2048_fence.txt 2>&1
timeout 120 python bench.py --steps 50 --warmup 5 --batch 2048 --no-cpu-baseline > gpurun_out/u_bench_fence_b2048.json 2>> gpurun_out/u_bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/u_bench_fence_cfg4.json 2>> gpurun_out/u_bench.err
cp /tmp/nofence.so paper_1611_09482_b200/libfastwavenet.so
