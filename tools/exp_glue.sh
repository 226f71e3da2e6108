#!/bin/bash
# Llama TP8 b64 ctx4k glue / pre-wait L2 prefetch experiment (one GPU)
set -u
OUT=gpurun_out/exp2; mkdir -p $OUT
for kb in 0 128 256 512 1024; do
  timeout 300 python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 --no-cpu-baseline --pre-wait-l2-kb $kb > $OUT/bench_llama4k_pre$kb.json 2> $OUT/bench_llama4k_pre$kb.err
  python -c "import json; d=json.load(open('$OUT/bench_llama4k_pre$kb.json')); print($kb, d['ms_per_step'], d['roofline']['frac'], d['roofline']['share_by_kind'])" >> $OUT/summary.txt 2>&1
done
timeout 300 python tools/trace_perop.py 8 64 --llama --context 4096 --pre-wait-l2-kb 512 > $OUT/trace_llama_pre512.txt 2>&1
