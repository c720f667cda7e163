#!/bin/bash
# session r03e: FFMA2 in the fp32 GEMVs (staged + small-batch kernels)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x -k "not tcgen05 and not cfg4 and not split" > gpurun_out/e_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/e_pytest.txt
for c in cfg1 cfg2_L14 cfg3 cfg5; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/e_bench_$c.json 2>> gpurun_out/e_bench.err; done
