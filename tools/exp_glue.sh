#!/bin/bash
set -u
OUT=gpurun_out/exp6; mkdir -p $OUT
for t in . _v2 . _v2; do
  (cd $t && timeout 600 python tools/sweep.py c4 2>/dev/null | head -3) >> $OUT/c4_ab.txt; echo "--- $t" >> $OUT/c4_ab.txt
  (cd $t && timeout 300 python bench.py --workload llama3-70b-tp8 --context 4096 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('llama', d['ms_per_step'])") >> $OUT/c4_ab.txt
done
