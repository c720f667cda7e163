#!/bin/bash
mkdir -p gpurun_out
for k in 1 2; do
timeout 1200 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 600 -k "simt_repeated" -rf > gpurun_out/x_pytest_simt_$k.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/x_pytest_simt_$k.txt
done
