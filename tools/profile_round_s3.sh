#!/bin/bash
# Round-2 session-3 measurement pass (GPU box, one GPU, repo root): GPU tests + smoke, the contract
# bench line and the reference arm, Llama TP8 lines (64k capacity-forced, 4k all-HBM), the tcgen05
# prefill sweep, C4 / C5 / Table 1 sweeps, the CTA-pair GEMM bench, the ncu launch list of one Llama 4k step, and one ncu --set full of
# the prefill kernel.
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --workload llama3-70b-tp8 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_llama64k.json 2> $OUT/bench_llama64k.err
timeout 600 python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_llama4k.json 2> $OUT/bench_llama4k.err
timeout 300 python tools/trace_perop.py 8 64 --llama --context 4096 > $OUT/trace_llama4k.txt 2>&1
timeout 600 python tools/prefill_bench.py > $OUT/prefill_bench.jsonl 2> $OUT/prefill_bench.err
timeout 900 python tools/sweep.py c4 > $OUT/c4.jsonl 2> $OUT/c4.err
timeout 900 python tools/sweep.py c5 > $OUT/c5.jsonl 2> $OUT/c5.err
timeout 900 python tools/sweep.py t1 > $OUT/t1.jsonl 2> $OUT/t1.err
timeout 600 python tools/pair_bench.py > $OUT/pair_bench.jsonl 2> $OUT/pair_bench.err
KF='regex:linear_kernel|umma_swap|splitk_reduce|split_attention|combine_kernel|embed|append_kernel|norm|residual|silu|rope|row_stats|prefill'
per() { python -c "import json,sys; d=json.load(open('$1')); print(d['gpu_launches']//d['steps'])"; }
PERL=$(per $OUT/bench_llama4k.json)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PERL * 4)) --launch-count $PERL --csv --log-file $OUT/launches_llama4k.csv \
  python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_llama4k.log 2>&1; echo "ncu llama rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill --launch-skip 3 --launch-count 1 \
  -o $OUT/prof_prefill python tools/prefill_bench.py 4 8192 2048 > $OUT/ncu_prefill.log 2>&1; echo "ncu prefill rc $?"
