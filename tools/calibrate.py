"""Run dak_calibrate (the congestion-control calibration sweep: the split GEMV timed at
each host-CTA count x window) and print its table and
choice as JSON lines: python tools/calibrate.py [chunk_bytes] [duration_us]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dur = int(sys.argv[2]) if len(sys.argv) > 2 else 300
n_host = (1, 2, 4, 8, 16)
window = tuple(w for w in (1, 2, 4, 6, 8) if 1024 + w * chunk <= 227 * 1024)
hbm = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
hp, dp = dak.host_alloc(256 << 20)
try:
    res, tab = dak.calibrate(hbm, hbm.numel(), dp, 256 << 20, n_host=n_host, window=window, chunk_bytes=chunk,
                             duration_us=dur, reps=3)
finally:
    dak.host_free(hp)
for i, n in enumerate(n_host):
    for j, w in enumerate(window):
        print(json.dumps(dict(n_host=n, window=w, inflight_kb=n * w * chunk // 1024, gemv_hbm_gbs=round(tab[i, j, 0] / 1e9, 1),
                              gemv_link_gbs=round(tab[i, j, 1] / 1e9, 2),
                              gemv_gbs=round((tab[i, j, 0] + tab[i, j, 1]) / 1e9, 1))))
print(json.dumps(dict(choice=res, chunk_bytes=chunk, duration_us=dur)))
