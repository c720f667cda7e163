#!/bin/bash
# round-2 GPU session W: full suite after the race fixes, every config's bench line, the
# reference arm, per-GPU loads, launch list
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/w_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/w_pytest.txt
python __graft_entry__.py > gpurun_out/w_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/w_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/w_bench_cfg4.json 2> gpurun_out/w_bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/w_ref_cfg4.json 2> gpurun_out/w_ref_cfg4.err
for b in 512 1024 2048 3072; do timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/w_bench_cfg4_b$b.json 2>> gpurun_out/w_sweep.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w_launches_cfg4.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:step_kernel -c 1 -o gpurun_out/w_step_app python tools/profile_step.py 10 cfg4 > gpurun_out/w_ncu_step.log 2>&1
