#!/bin/bash
set -u
OUT=gpurun_out/exp13; mkdir -p $OUT
timeout 300 python tools/trace_perop.py 8 64 --llama --context 4096 > $OUT/trace_llama.txt 2>&1
