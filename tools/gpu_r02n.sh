#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/trace_chain.py --batch 512 > gpurun_out/n_trace_split.txt 2>&1
FW_CHAIN_SPLIT=0 timeout 120 python tools/trace_chain.py --batch 512 > gpurun_out/n_trace_nosplit.txt 2>&1
