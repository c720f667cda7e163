#!/bin/bash
# session r03j: the warp-MMA kernel in the default dispatch -- full GPU suite + benches
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/j_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/j_pytest.txt
python __graft_entry__.py > gpurun_out/j_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/j_smoke.txt
for c in cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/j_bench_$c.json 2> gpurun_out/j_bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches_cfg5.csv python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_hmma_kernel -c 1 -o gpurun_out/j_hmma_cfg5 python tools/profile_step.py 10 cfg5 > gpurun_out/j_ncu.log 2>&1
