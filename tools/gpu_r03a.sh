#!/bin/bash
# session r03a: HEAD after the compile-time specialisations -- full GPU suite, smoke,
# every config's bench line, reference arm, launch list, ncu of the specialised kernels
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/a_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.txt
python __graft_entry__.py > gpurun_out/a_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/a_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/a_bench_cfg4.json 2> gpurun_out/a_bench_cfg4.err
for c in cfg1 cfg2_L14 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/a_bench_$c.json 2> gpurun_out/a_bench_$c.err; done
timeout 600 python tools/depth_sweep.py --steps 1000 --naive-steps 20 > gpurun_out/a_depth_sweep.jsonl 2> gpurun_out/a_depth_sweep.err
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/a_lat_cfg1 python tools/profile_step.py 50 cfg1 > gpurun_out/a_ncu.log 2>&1
timeout 900 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_lat_kernel -c 1 -o gpurun_out/a_lat_cfg3 python tools/profile_step.py 10 cfg3 >> gpurun_out/a_ncu.log 2>&1
timeout 900 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_staged_kernel -c 1 -o gpurun_out/a_staged_cfg5 python tools/profile_step.py 10 cfg5 >> gpurun_out/a_ncu.log 2>&1
