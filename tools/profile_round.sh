#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root, one GPU):
#   bench lines (OPT-30B b8 = the contract line, Llama-3-70B TP8 shard b64), the reference arm, an
#   ncu launch list of ONE timed decode step of each workload with per-launch DRAM bytes (-> the
#   per-workload linear_traffic_<workload>.json bench.py reads), a --set full capture of the
#   dominant kernel inside the step, and the link-counter cases (tools/link_counters.py).
# The bench runs: eager warm step, W warm-up replays, K timed replays, K e2e replays, the in-step
# trace replays -> with --steps 1 --warmup 3, skipping 4 steps lands on the first timed one.
set -u
R=${1:-r02}
OUT=gpurun_out/$R
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc $?"
python bench.py --workload llama3-70b-tp8 --steps 10 --warmup 3 > $OUT/bench_llama.json 2> $OUT/bench_llama.err; echo "llama rc $?"
KF='regex:linear_kernel|umma_swap|splitk_reduce|split_attention|combine_kernel|embed|append_kernel|norm|residual|silu|rope|row_stats|prefill'
per() { python -c "import json,sys; d=json.load(open('$1')); print(d['gpu_launches']//d['steps'])"; }
PER=$(per $OUT/bench.json)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PER * 4)) --launch-count $PER --csv --log-file $OUT/launches_opt.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_opt.log 2>&1; echo "ncu opt rc $?"
PERL=$(per $OUT/bench_llama.json)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PERL * 4)) --launch-count $PERL --csv --log-file $OUT/launches_llama.csv \
  python bench.py --workload llama3-70b-tp8 --steps 1 --warmup 3 > $OUT/ncu_launch_llama.log 2>&1; echo "ncu llama rc $?"
# full capture: layer 1's linears inside the timed OPT step (qkv, o, fc1, fc2)
LIN=$((4 * 48 + 1))
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:split_linear \
  --launch-skip $(( LIN * 4 + 4 )) --launch-count 4 -o $OUT/prof_linear \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1; echo "ncu full rc $?"
# link counters: one launch per case
python tools/link_counters.py > $OUT/link_cases.jsonl 2> $OUT/link_cases.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem.sum \
  --clock-control none -k 'regex:split_linear|umma_linear|umma_swap|split_attention' --csv --log-file $OUT/link_ncu.csv \
  python tools/link_counters.py > $OUT/link_ncu.log 2>&1; echo "ncu link rc $?"
