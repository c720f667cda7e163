#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "cfg5 or staged" > gpurun_out/z_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/z_pytest.txt
timeout 300 python bench.py --config cfg5 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/z_bench_cfg5.json 2>> gpurun_out/z_bench.err
FW_LAT_GENERIC=1 timeout 300 python bench.py --config cfg5 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/z_bench_cfg5_generic.json 2>> gpurun_out/z_bench.err
