#!/bin/bash
# session r03f: warp-MMA kernel for the fp32 configs -- parity and timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -q -p no:cacheprovider --timeout 600 -x -k "cfg5 or cfg3" -rf > gpurun_out/f_pytest_long.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/f_pytest_long.txt
for c in cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/f_bench_$c.json 2>> gpurun_out/f_bench.err
  FW_HMMA_NT=2 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/f_bench_${c}_nt2.json 2>> gpurun_out/f_bench.err
done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "not tcgen05 and not cfg4 and not split" -rf > gpurun_out/f_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/f_pytest.txt
