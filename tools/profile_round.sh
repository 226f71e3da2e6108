#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root, one GPU):
#   bench line (+ cpu_baseline), reference arm, ncu launch list of ONE timed decode step with
#   per-launch DRAM bytes, and a --set full capture of the dominant kernels (q and fc1 linears).
# Kernel launches per step (per-op path, fused pre-norm, fused QKV, KV append fused into attention): 1 embed + 48 x (qkv,
# attention, o, fc1, fc2) + head = 242. The bench runs: eager warm step, 3 warm-up replays, K timed replays,
# K e2e replays, then the per-launch roofline loop -> skip 4 steps to land on the first timed one.
set -u
R=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 20 --warmup 3 > $OUT/bench_$R.json 2> $OUT/bench_$R.err; echo "bench rc $?"
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$R.json 2> $OUT/bench_ref_$R.err; echo "ref rc $?"
PER=$(python -c "from paper_2604_26074_b200.engine import OPT_30B; print(1 + 5 * OPT_30B.n_layers + 1)")
LIN=$(python -c "from paper_2604_26074_b200.engine import OPT_30B; print(4 * OPT_30B.n_layers + 1)")
KF='regex:split_linear|split_attention|combine_kernel|embed_kernel|append_kernel|layernorm_kernel'
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KF" --launch-skip $((PER * 4)) --launch-count $PER --csv --log-file $OUT/launches_$R.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$R.log 2>&1; echo "ncu list rc $?"
# full capture: layer 1's linears inside the timed step (qkv, o, fc1, fc2)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:split_linear \
  --launch-skip $(( LIN * 4 + 4 )) --launch-count 4 -o $OUT/prof_linear_$R \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$R.log 2>&1; echo "ncu full rc $?"
# full capture: layer 1's split attention inside the timed step
ATT=$(python -c "from paper_2604_26074_b200.engine import OPT_30B; print(OPT_30B.n_layers)")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_attention \
  --launch-skip $(( ATT * 4 + 1 )) --launch-count 1 -o $OUT/prof_attn_$R \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_attn_$R.log 2>&1; echo "ncu attn rc $?"
