#!/bin/bash
# round-2 GPU session B: tests, bench lines for every config, ncu captures (application
# replay keeps the step kernel's cluster dimension), prefill launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/b_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/b_pytest.txt
python __graft_entry__.py > gpurun_out/b_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/b_smoke.txt
for c in cfg5 cfg3 cfg1; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --cpu-seconds 10 > gpurun_out/b_bench_$c.json 2> gpurun_out/b_bench_$c.err
done
timeout 300 python tools/profile_prefill.py cfg5 64 > gpurun_out/b_prefill_cfg5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches_prefill_cfg5.csv python tools/profile_prefill.py cfg5 64 > /dev/null 2>&1
timeout 1500 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:step_kernel -c 1 -o gpurun_out/b_step_app python tools/profile_step.py 10 cfg4 > gpurun_out/b_ncu_step.log 2>&1
timeout 900 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:cell_cluster_kernel -c 1 -o gpurun_out/b_cluster_app python tools/profile_step.py 20 cfg1 > gpurun_out/b_ncu_cluster.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cell_staged_kernel -s 1 -c 1 -o gpurun_out/b_staged_cfg3 python tools/profile_step.py 10 cfg3 > gpurun_out/b_ncu_staged.log 2>&1
