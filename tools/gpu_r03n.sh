#!/bin/bash
# session r03n: committed state -- every config's bench line (CPU baselines included), the
# reference arm, cfg5 launch list + ncu of the warp-MMA kernel, depth sweep
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/n_bench_cfg4.json 2> gpurun_out/n_bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/n_ref_cfg4.json 2> gpurun_out/n_ref_cfg4.err
for c in cfg1 cfg2_L14 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/n_bench_$c.json 2> gpurun_out/n_bench_$c.err; done
FW_SIMT_HMMA=0 timeout 900 python bench.py --config cfg5 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/n_bench_cfg5_staged.json 2>/dev/null
for b in 512 1024 2048; do timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/n_bench_cfg4_b$b.json 2>> gpurun_out/n_sweep.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launches_cfg5.csv python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_hmma_kernel -c 1 -o gpurun_out/n_hmma_cfg5 python tools/profile_step.py 10 cfg5 > gpurun_out/n_ncu.log 2>&1
timeout 120 python tools/trace_hmma.py cfg5 > gpurun_out/n_trace_hmma.txt 2>&1
