#!/bin/bash
# session r03s: the final state -- full GPU suite, smoke, bench lines with the unmodified
# reference's proxy timing (baseline/_ref), reference arm
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/s_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/s_pytest.txt
python __graft_entry__.py > gpurun_out/s_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/s_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s_bench_cfg4.json 2> gpurun_out/s_bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s_ref_cfg4.json 2> gpurun_out/s_ref_cfg4.err
for c in cfg1 cfg2_L14 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 10 > gpurun_out/s_bench_$c.json 2> gpurun_out/s_bench_$c.err; done
