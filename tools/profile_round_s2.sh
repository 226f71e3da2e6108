#!/bin/bash
# Round-2 second-session measurement pass (run on the GPU box from the repo root, one GPU):
# GPU tests + smoke, the contract bench line and the reference arm, Llama TP8 64k and 4k, the C2
# sweep, the ncu launch lists of one timed step (-> per-workload traffic files), a --set full of the
# swapped tcgen05 [gate; up] GEMM inside the Llama 4k step, C1 per-launch vs chain.
set -u
OUT=gpurun_out/r02b
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --workload llama3-70b-tp8 --steps 10 --warmup 3 > $OUT/bench_llama.json 2> $OUT/bench_llama.err
timeout 600 python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 > $OUT/bench_llama4k.json 2> $OUT/bench_llama4k.err
bash tools/c2_sweep.sh r02b > $OUT/c2_summary.txt 2>&1
for a in "512 16" "512 16 indep=1" "512 16 tau_us=1.5 indep=1"; do timeout 120 python tools/c1_chain.py $a >> $OUT/c1_chain.jsonl 2>&1; done
KF='regex:linear_kernel|umma_swap|splitk_reduce|split_attention|combine_kernel|embed|append_kernel|norm|residual|silu|rope|row_stats|prefill'
per() { python -c "import json,sys; d=json.load(open('$1')); print(d['gpu_launches']//d['steps'])"; }
PER=$(per $OUT/bench.json)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PER * 4)) --launch-count $PER --csv --log-file $OUT/launches_opt.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_opt.log 2>&1; echo "ncu opt rc $?"
PERL=$(per $OUT/bench_llama4k.json)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PERL * 4)) --launch-count $PERL --csv --log-file $OUT/launches_llama4k.csv \
  python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 > $OUT/ncu_launch_llama4k.log 2>&1; echo "ncu llama rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_swap --launch-skip 40 --launch-count 3 \
  -o $OUT/prof_swap python bench.py --workload llama3-70b-tp8 --context 4096 --steps 1 --warmup 3 > $OUT/ncu_swap.log 2>&1; echo "swap rc $?"
