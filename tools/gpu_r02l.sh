#!/bin/bash
# round-2 GPU session L: the committed state -- tests, every config's bench line, the
# reference arm, per-GPU strong-scaling loads, depth sweep, prefill, ncu evidence
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/l_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l_pytest.txt
python __graft_entry__.py > gpurun_out/l_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/l_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/l_bench_cfg4.json 2> gpurun_out/l_bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/l_ref_cfg4.json 2> gpurun_out/l_ref_cfg4.err
for c in cfg1 cfg2_L14 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/l_bench_$c.json 2> gpurun_out/l_bench_$c.err; done
for b in 512 1024 2048; do timeout 300 python bench.py --steps 50 --warmup 5 --batch $b --no-cpu-baseline > gpurun_out/l_bench_cfg4_b$b.json 2>> gpurun_out/l_sweep.err; done
timeout 600 python tools/depth_sweep.py --steps 1000 --naive-steps 20 > gpurun_out/l_depth_sweep.jsonl 2> gpurun_out/l_depth_sweep.err
for c in "cfg5 64" "cfg3 500" "cfg1 2000"; do timeout 300 python tools/profile_prefill.py $c >> gpurun_out/l_prefill.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches_prefill_cfg5.csv python tools/profile_prefill.py cfg5 64 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches_cfg4.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/l_lat_cfg1 python tools/profile_step.py 50 cfg1 > gpurun_out/l_ncu.log 2>&1
timeout 900 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/l_lat_cfg3 python tools/profile_step.py 10 cfg3 >> gpurun_out/l_ncu.log 2>&1
timeout 900 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_staged_kernel -c 1 -o gpurun_out/l_staged_cfg5 python tools/profile_step.py 10 cfg5 >> gpurun_out/l_ncu.log 2>&1
