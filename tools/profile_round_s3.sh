#!/bin/bash
# Round-2 session-3 validation pass (GPU box, one GPU, repo root): GPU tests + smoke, the contract
# bench line, the tcgen05 prefill sweep, and one ncu --set full capture of the prefill kernel.
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 python tools/prefill_bench.py > $OUT/prefill_bench.jsonl 2> $OUT/prefill_bench.err; echo "prefill rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill --launch-skip 3 --launch-count 1 \
  -o $OUT/prof_prefill python tools/prefill_bench.py 4 8192 2048 > $OUT/ncu_prefill.log 2>&1; echo "ncu prefill rc $?"
