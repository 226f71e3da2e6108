"""Trace one persistent decode step (dak_step globaltimer stamps per op per CTA) and summarise
where the step's time goes: per-op critical-path increment, dependency hand-off latency, spread
between the first and the last CTA to finish (host-tier CTA vs HBM CTAs)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402
from paper_2604_26074_b200.engine import DakOPT, HW, OPTConfig  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = OPTConfig(n_layers=layers)
eng = DakOPT(cfg, batch, 64, HW(hbm_bps=6555.5e9, link_bps=51.5e9), mode=dak.PLAN_BALANCED, fused_qkv=False)
eng.enable_persistent_step()
plan = eng.step_plan
G, n_ops = plan.grid, plan.n_ops
tr = torch.zeros(n_ops * G * 4, dtype=torch.int64, device="cuda")
for _ in range(3):
    eng.enqueue_step()
torch.cuda.synchronize()
plan.trace = tr.data_ptr()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.enqueue_step()
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
T = tr.cpu().numpy().reshape(n_ops, G, 4).astype(np.float64)
names = []
for i, o in enumerate(eng.step_ops):
    names.append({0: "embed", 1: "ln", 2: "linear", 3: "attn", 4: "combine"}[o.type] + (f"[M={o.M}]" if o.type == 2 else ""))
t0 = T[T > 0].min()
T = np.where(T > 0, T - t0, np.nan)
rows = []
prev_end = 0.0
for i in range(n_ops):
    done = T[i, :, 3]
    dep = T[i, :, 1]
    first = T[i, :, 2]
    end = np.nanmax(done)
    rows.append(dict(op=i, name=names[i], end_us=round(end / 1e3, 2), inc_us=round((end - prev_end) / 1e3, 2),
                     dep_seen_min_us=round(np.nanmin(dep) / 1e3, 2) if np.isfinite(np.nanmin(dep)) else None,
                     first_stage_med_us=round(np.nanmedian(first) / 1e3, 2) if np.any(np.isfinite(first)) else None,
                     done_spread_us=round((np.nanmax(done) - np.nanmin(done)) / 1e3, 2),
                     host_cta_done_us=round(done[0] / 1e3, 2), median_done_us=round(np.nanmedian(done) / 1e3, 2)))
    prev_end = end
agg = {}
for r in rows:
    k = r["name"]
    a = agg.setdefault(k, dict(n=0, inc=0.0, spread=0.0))
    a["n"] += 1
    a["inc"] += r["inc_us"]
    a["spread"] += r["done_spread_us"]
print(json.dumps(dict(layers=layers, step_ms=step_ms, ops=n_ops, grid=G, ring_bytes=plan.ring_bytes,
                      bytes=eng.bytes_per_step()["total"], gbs=eng.bytes_per_step()["total"] / step_ms / 1e6)))
for k, a in agg.items():
    print(json.dumps(dict(kind=k, count=a["n"], total_inc_us=round(a["inc"], 1), mean_inc_us=round(a["inc"] / a["n"], 2),
                          mean_done_spread_us=round(a["spread"] / a["n"], 2))))
for r in rows[:40]:
    print(json.dumps(r))
eng.close()
