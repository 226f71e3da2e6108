"""Per-op launch timeline of the per-op decode step (dak_layer path) from dak_trace stamps.

Usage: python tools/trace_perop.py [layers] [batch] [--no-fuse-norm] [--no-pdl]
       python tools/trace_perop.py [layers] [batch] --llama [--context N]   (Llama-3-70B TP8 rank shard,
       HBM only, 1-rank NCCL communicator, as bench.py --workload llama3-70b-tp8)
Captures one decode step in a CUDA graph with tracing on, replays it, and prints per launch the
CTA start spread, the dependency-release time, the first-stage time and the completion time
(all relative to the step's first stamp), then per-kind aggregates of the incremental time
(this op's last CTA done minus the previous op's last CTA done).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2604_26074_b200 import dak
from paper_2604_26074_b200.engine import DakOPT, HW, OPTConfig, OPT_30B


def main():
    args = [a for i, a in enumerate(sys.argv[1:], 1) if not a.startswith("--") and sys.argv[i - 1] != "--context"]
    layers = int(args[0]) if args else 8
    batch = int(args[1]) if len(args) > 1 else 8
    # the bench's planner rates (the C5 sweep's sustained HBM / link rates), so the plan matches bench.py
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    ph, pl, _ = bench.planner_rates(6555.5, 51.5)
    hw = HW(hbm_bps=ph * 1e9, link_bps=pl * 1e9)
    if "--llama" in sys.argv:
        from dataclasses import replace
        from paper_2604_26074_b200.llama import DakLlama, LLAMA3_70B
        ctx = int(sys.argv[sys.argv.index("--context") + 1]) if "--context" in sys.argv else 4096
        comm = dak.comm_init(dak.comm_unique_id(), 0, 1)
        eng = DakLlama(replace(LLAMA3_70B, n_layers=layers), batch, ctx, hw, tp_rank=0, tp_size=8, comm=comm,
                       mode=dak.PLAN_EXACT, y_req=0, pdl="--no-pdl" not in sys.argv)
    else:
        cfg = OPT_30B if layers == 48 else OPTConfig(n_layers=layers)
        eng = DakOPT(cfg, batch, 64, hw, mode=dak.PLAN_BALANCED, fuse_norm="--no-fuse-norm" not in sys.argv,
                     pdl="--no-pdl" not in sys.argv)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eng.enqueue_step(s)
    s.synchronize()
    n_launch = eng.kernels_per_step() + 8
    buf = torch.zeros(n_launch * 1024 * 4, dtype=torch.int64, device="cuda")
    dak.trace_enable(buf, n_launch)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        eng.enqueue_step(s)
    meta = dak.trace_launches()
    dak.trace_enable(None, 0)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    g.replay()
    ev1.record(s)
    torch.cuda.synchronize()
    step_ms = ev0.elapsed_time(ev1)
    T = buf.view(-1, 1024, 4).cpu().numpy().astype(np.float64)
    rows = []
    t0 = None
    for i, m in enumerate(meta):
        st = T[i, :m["grid"]]
        valid = st[:, 0] > 0
        s0 = st[valid, 0]
        if t0 is None:
            t0 = s0.min()
        end = st[valid, 3].max()
        dep = st[valid, 1][st[valid, 1] > 0]
        fs = st[valid, 2][st[valid, 2] > 0]
        rows.append(dict(i=i, kind=m["kind"], a=m["a"], b=m["b"], grid=m["grid"],
                         start_min=(s0.min() - t0) / 1e3, start_max=(s0.max() - t0) / 1e3,
                         dep_max=((dep.max() - t0) / 1e3) if dep.size else None,
                         first_stage_med=((np.median(fs) - t0) / 1e3) if fs.size else None,
                         end_max=(end - t0) / 1e3))
    prev_end = 0.0
    agg = {}
    for r in rows:
        inc = r["end_max"] - prev_end
        r["inc"] = inc
        prev_end = r["end_max"]
        key = r["kind"] + (f"[M={r['a']}]" if r["kind"] == "linear" else "")
        a = agg.setdefault(key, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += inc
        a[2] += r["end_max"] - r["start_min"]
        a[3] += (r["end_max"] - r["dep_max"]) if r["dep_max"] is not None else 0.0
    print(json.dumps(dict(layers=layers, batch=batch, step_ms_graph=step_ms, traced_span_us=prev_end,
                          launches=len(rows))))
    for k, (c, inc, dur, after_dep) in agg.items():
        print(json.dumps(dict(kind=k, count=c, total_inc_us=round(inc, 1), mean_inc_us=round(inc / c, 2),
                              mean_span_us=round(dur / c, 2), mean_after_dep_us=round(after_dep / c, 2))))
    # attention per-CTA phases: dep -> first unit done, then time per further unit
    for i, m in enumerate(meta):
        if m["kind"] != "attention":
            continue
        st = T[i, :m["grid"]]
        ok = (st[:, 0] > 0) & (st[:, 2] > 0)
        first = (st[ok, 2] - st[ok, 1]) / 1e3
        rest = (st[ok, 3] - st[ok, 2]) / 1e3
        print(json.dumps(dict(attention_launch=i, ctas_with_units=int(ok.sum()),
                              dep_to_first_unit_us=[round(float(np.percentile(first, q)), 2) for q in (0, 50, 100)],
                              after_first_unit_us=[round(float(np.percentile(rest, q)), 2) for q in (0, 50, 100)],
                              start_to_dep_us=[round(float(np.percentile((st[ok, 1] - st[ok, 0]) / 1e3, q)), 2)
                                               for q in (0, 50, 100)])))
        break
    # linear: host vs HBM CTA completion
    for i, m in enumerate(meta):
        if m["kind"] != "linear":
            continue
        st = T[i, :m["grid"]]
        e = st[:, 3]
        print(json.dumps(dict(linear_launch=i, M=m["a"], end_spread_us=round(float((e.max() - np.median(e)) / 1e3), 2),
                              first2_end_minus_median_us=round(float((e[:2].max() - np.median(e)) / 1e3), 2),
                              start_spread_us=round(float((st[:, 0].max() - st[:, 0].min()) / 1e3), 2),
                              dep_to_first_stage_med_us=round(float(np.median(st[:, 2] - st[:, 1]) / 1e3), 2),
                              first_stage_to_end_med_us=round(float(np.median(st[:, 3] - st[:, 2]) / 1e3), 2))))
        if i > 20:
            break
    mid = len(rows) // 2
    for r in rows[mid - 6: mid + 8]:
        print(" ".join(f"{k}={v:.2f}" if isinstance(v, float) else f"{k}={v}" for k, v in r.items()))
    eng.close()


if __name__ == "__main__":
    main()
