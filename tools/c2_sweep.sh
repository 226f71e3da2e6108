#!/bin/bash
# BASELINE configs[1] sweep: OPT-30B decode step at batch 1, 2, 4, 8, 16 (BALANCED
# plan, r*), and at batch 8 with the global ratio forced to R = 0.05 / 0.1 / 0.2 / 0.4 (EXACT plan,
# the paper's sweep shape P:L697-704). One bench.py JSON line per point -> profiles/<round>/c2_sweep.jsonl
set -u
R=${1:-r02}
OUT=gpurun_out/$R
mkdir -p $OUT
: > $OUT/c2_sweep.jsonl
for b in 1 2 4 16; do
  python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline >> $OUT/c2_sweep.jsonl 2>> $OUT/c2_sweep.err
done
for r in 0.05 0.1 0.2 0.4; do
  python bench.py --batch 8 --ratio $r --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/c2_sweep.jsonl 2>> $OUT/c2_sweep.err
done
python - "$R" <<'PY'
import json
import sys
for l in open("gpurun_out/%s/c2_sweep.jsonl" % sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02/c2_sweep.jsonl"):
    d = json.loads(l)
    c, rf = d["config"], d["roofline"]
    print(c["batch"], c["plan"], "r=%.4f" % c["host_ratio"], "%.3f ms" % d["ms_per_step"], "%.0f GB/s" % d["value"],
          "tok/s %.0f" % d["tokens_per_s"], "EB(r) %.0f" % rf["split_roofline_gbs"], "frac %.3f" % rf["step_frac_of_split_roofline"])
PY
