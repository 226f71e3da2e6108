"""C5-style host-ratio sweep on the tcgen05 split-K path (batch 64, swapped operands): the Llama TP8
[gate; up] shard 7168 x 8192 at r in {0, r*, 2%, 5%, 20%, 50%}; fraction of EB(r) (development tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_linear import time_cfg  # noqa: E402
from tools.sweep import eb, peaks  # noqa: E402

bg, bl = peaks()
M, K, N = 7168, 8192, 64
for r in (0.0, bl / (bg + bl), 0.02, 0.05, 0.2, 0.5):
    h = int(round(r * M / 128)) * 128
    res = time_cfg(M, K, N, h, 64, launches=16 if h > M // 8 else 64, reps=3, pdl=1, ws=True)
    rr = h / M
    g = res["hbm_gbs"] + res["host_gbs"]
    print(json.dumps(dict(M=M, K=K, N=N, r=round(rr, 4), us=round(res["us"], 1), gbs=round(g, 1),
                          host_gbs=round(res["host_gbs"], 2), frac=round(g * 1e9 / eb(rr, bg, bl), 4),
                          grid=res["info"]["grid"])), flush=True)
