#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/y_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/y_pytest.txt
python __graft_entry__.py > gpurun_out/y_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/y_smoke.txt
timeout 900 python bench.py > gpurun_out/y_bench_default.json 2> gpurun_out/y_bench_default.err
