#!/bin/bash
# Llama TP8 b64 ctx4k glue-kernel experiment (one GPU): parity of the touched kernels, per-op trace, bench lines
set -u
OUT=gpurun_out/exp3; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_llama.py tests/test_gpu_engine.py tests/test_gpu_edges.py tests/test_gpu_tp_multi.py -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc $?" >> $OUT/pytest.txt
timeout 300 python tools/trace_perop.py 8 64 --llama --context 4096 > $OUT/trace_llama.txt 2>&1
timeout 300 python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_llama4k.json 2> $OUT/bench_llama4k.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_opt.json 2> $OUT/bench_opt.err
