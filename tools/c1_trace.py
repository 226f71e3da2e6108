"""Where the time of a chained C1 GEMV goes (BASELINE configs[0]: 4096 x 4096 bf16, N = 1, host
share at the planner's r*): a CUDA graph of back-to-back dak_linear launches (PDL, distinct weight
copies > 4 x L2) traced with the library's per-CTA globaltimer stamps. Prints, per launch and as
medians: the gap from the previous launch's last CTA end to this launch's first CTA start, the
dependency wait, the first consumed stage, and the CTA end spread -- plus the chained time per
launch from CUDA events.

  python tools/c1_trace.py [kc] [launches]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402
from tools.bench_linear import setup  # noqa: E402


def main():
    kc = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
    extra = dict(kv.split("=") for kv in sys.argv[3:])
    pf_mb = float(extra.pop("pf_mb", 0))  # L2 warm-up of the NEXT launch's weights (dak_linear_args.l2_prefetch)
    tau_us = float(extra.pop("tau_us", 0))  # latency-aware planner: host link latency (dak_hw.host_latency_s)
    h_force = int(extra.pop("h", -1))       # host rows override (-1: the planner's)
    cfg = dict(pdl=1, congestion_control=1, **{k: int(v) for k, v in extra.items()})
    M = K = 4096
    N = 1
    plan, _ = dak.plan_ratios(dict(hbm_bps=6542.1e9, link_bps=51.5e9, host_latency_s=tau_us * 1e-6),
                              [dict(n_units=M // 16, unit_bytes=16 * K * 2, total_bytes=M * K * 2, T=0.0)], 0,
                              dak.PLAN_BALANCED)
    h = plan[0]["host_units"] * 16 if h_force < 0 else h_force
    copies = 24
    hbm, hosts, x, y = setup(M, K, N, h, kc, copies)
    pf = int(pf_mb * (1 << 20)) // 16 * 16
    args = [dak.linear_args(hosts[i % copies][1] if h else None, hbm[i % copies], M, K, h, kc, N, x, y, cfg=cfg,
                            l2_prefetch=hbm[(i + 1) % copies] if pf else None, l2_prefetch_bytes=pf)
            for i in range(n)]
    info = dak.linear_query(args[0])
    s = torch.cuda.Stream()
    buf = torch.zeros(n * 1024 * 4, dtype=torch.int64, device="cuda")
    with torch.cuda.stream(s):
        for a in args[:4]:
            dak.linear(a, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for a in args:
                dak.linear(a, s)
        dak.trace_enable(buf, n)
        gt = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gt, stream=s):
            for a in args:
                dak.linear(a, s)
        dak.trace_enable(None, 0)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(s)
        with torch.cuda.stream(s):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    gt.replay()
    torch.cuda.synchronize()
    T = buf.view(n, 1024, 4).cpu().numpy().astype(np.float64)[:, :info["grid"]]
    rows = []
    prev_end = None
    for i in range(n):
        st = T[i]
        start, dep, first, end = st[:, 0], st[:, 1], st[:, 2], st[:, 3]
        r = dict(start_gap=(start.min() - prev_end) / 1e3 if prev_end else None,
                 start_spread=(start.max() - start.min()) / 1e3,
                 dep_after_start=(np.median(dep[dep > 0]) - start.min()) / 1e3 if (dep > 0).any() else None,
                 first_stage_after_start=(np.median(first[first > 0]) - start.min()) / 1e3 if (first > 0).any() else None,
                 end_after_start_med=(np.median(end) - start.min()) / 1e3, end_after_start_max=(end.max() - start.min()) / 1e3,
                 host_end_after_start=(end[:info["n_cta_host"]].max() - start.min()) / 1e3 if info["n_cta_host"] else None,
                 inc=(end.max() - prev_end) / 1e3 if prev_end else None)
        prev_end = end.max()
        rows.append(r)
    med = {k: round(float(np.median([r[k] for r in rows[4:] if r[k] is not None])), 3) for k in rows[4]}
    print(json.dumps(dict(kc=kc, h=h, tau_us=tau_us, pf_mb=pf_mb, grid=info["grid"], n_cta_host=info["n_cta_host"], stages=info["stages_hbm"],
                          smem=info["smem_bytes"], path=info["path"], us_per_launch_events=round(float(np.median(ts)), 3),
                          gbs=round(M * K * 2 / (np.median(ts) * 1e-6) / 1e9, 1), medians_us=med)))
    for i, h_ in enumerate(hosts):
        dak.host_free(h_[0])


if __name__ == "__main__":
    main()
