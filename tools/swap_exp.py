"""tcgen05 split-K at the Llama-3-70B TP8 rank-shard shapes, b64: weight rows as the MMA's M
(force_path 3) vs swapped operands (force_path 4, umma_swap_kernel). 64 chained launches + the
split-K reduce each, PDL, graph-replayed."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_linear import time_cfg  # noqa: E402

for (M, K) in ((1280, 8192), (8192, 1024), (7168, 8192), (8192, 3584)):
    for fp in (3, 4):
        r = time_cfg(M, K, 64, 0, 64, pdl=1, force_path=fp, ws=True)
        print(json.dumps(dict(M=M, K=K, N=64, force_path=fp, us=round(r["us"], 2), gbs=round(r["gbs"], 1),
                              grid=r["info"]["grid"], stages=r["info"]["stages_hbm"])), flush=True)
