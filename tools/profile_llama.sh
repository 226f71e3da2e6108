#!/bin/bash
# Llama-3-70B TP8 shard b64, 4k context, all in HBM (the C3 family's large-batch tcgen05 path):
# launch list of one timed step + --set full of the step's [gate; up] swap-GEMM and attention.
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 > $OUT/llama4k.json 2> $OUT/llama4k.err
PER=$(python -c "import json; d=json.load(open('$OUT/llama4k.json')); print(d['gpu_launches']//d['steps'])")
KF='regex:linear_kernel|umma_swap|splitk_reduce|split_attention|combine_kernel|embed|append_kernel|norm|residual|silu|rope|row_stats'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none \
  -k "$KF" --launch-skip $((PER * 4)) --launch-count $PER --csv --log-file $OUT/launches_llama4k.csv \
  python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 > $OUT/ncu_llama4k.log 2>&1; echo "list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_swap --launch-skip 40 --launch-count 3 \
  -o $OUT/prof_swap python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 > $OUT/ncu_swap.log 2>&1; echo "swap rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_attention --launch-skip 10 --launch-count 1 \
  -o $OUT/prof_attn_llama python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 > $OUT/ncu_attn.log 2>&1; echo "attn rc $?"
