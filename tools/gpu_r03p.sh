#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg5 --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/p_bench_cfg5.json 2> gpurun_out/p_bench_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_cfg5.csv python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_hmma_kernel -c 1 -o gpurun_out/p_hmma_cfg5 python tools/profile_step.py 10 cfg5 > gpurun_out/p_ncu.log 2>&1
timeout 120 python tools/trace_hmma.py cfg5 > gpurun_out/p_trace_hmma.txt 2>&1
