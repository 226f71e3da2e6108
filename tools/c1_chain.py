"""C1 (4096 x 4096 bf16 GEMV, N = 1, host rows at the planner's r*) as a DEPENDENT chain: x of op i
is y of op i-1, 16 distinct weight copies (> 4 x L2). Times (a) 16 dak_linear launches (PDL) and (b)
one dak_linear_chain launch of the 16 ops, both replayed as CUDA graphs; prints us per op and GB/s
(weights + x + y bytes) and the fraction of the split roofline EB(r) = 1 / max((1-r)/B_g, r/B_l).

  python tools/c1_chain.py [kc] [n_ops] [key=value cfg ...]   (e.g. n_cta_host=2 tau_us=1.5)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402


def main():
    kc = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    extra = dict(kv.split("=") for kv in sys.argv[3:])
    tau_us = float(extra.pop("tau_us", 0))
    h_force = int(extra.pop("h", -1))
    indep = int(extra.pop("indep", 0))  # 1: independent ops (one x, a y per op): steady-state operator throughput
    M = K = int(extra.pop("M", 4096))
    N = int(extra.pop("N", 1))
    cfg = dict(pdl=1, congestion_control=1, force_path=2, **{k: int(v) for k, v in extra.items()})
    Bg, Bl = 6542.1e9, 51.5e9
    plan, _ = dak.plan_ratios(dict(hbm_bps=Bg, link_bps=Bl, host_latency_s=tau_us * 1e-6),
                              [dict(n_units=M // 16, unit_bytes=16 * K * 2, total_bytes=M * K * 2, T=0.0)], 0,
                              dak.PLAN_BALANCED)
    h = plan[0]["host_units"] * 16 if h_force < 0 else h_force
    hbm = [torch.empty((M - h) * K, device="cuda", dtype=torch.bfloat16).normal_() for _ in range(L)]
    hosts = [dak.host_alloc(max(h * K * 2, 16)) for _ in range(L)]
    xs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.01, torch.zeros(N, K, device="cuda", dtype=torch.bfloat16)]
    ys = [torch.zeros(N, M, device="cuda", dtype=torch.bfloat16) for _ in range(L)]
    ops = [dak.linear_args(hosts[i][1] if h else None, hbm[i], M, K, h, kc, N, xs[0] if indep else xs[i % 2],
                           ys[i] if indep else xs[(i + 1) % 2], cfg=cfg) for i in range(L)]
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()

    def timed(enqueue, reps=5, per_graph=8):
        with torch.cuda.stream(s):
            enqueue()
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(per_graph):
                    enqueue()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            e0.record(s)
            with torch.cuda.stream(s):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3 / (per_graph * L))
        return float(np.median(ts))

    t_single = timed(lambda: [dak.linear(a, s) for a in ops])
    t_chain = timed(lambda: dak.linear_chain(ops, ws, ws.numel(), s))
    r = h / M
    eb = 1.0 / max((1 - r) / Bg, r / Bl)
    nbytes = M * K * 2 + 2 * N * K * 2
    out = dict(kc=kc, h=h, r=round(r, 5), n_ops=L, chain="independent" if indep else "dependent (x of op i = y of op i-1)",
               tau_us=tau_us, cfg=cfg, eb_gbs=round(eb / 1e9, 1))
    for name, t in (("launches", t_single), ("chain", t_chain)):
        out[name] = dict(us_per_op=round(t * 1e6, 3), gbs=round(nbytes / t / 1e9, 1), frac_eb=round(nbytes / t / eb, 3))
    print(json.dumps(out))
    for hp, _ in hosts:
        dak.host_free(hp)


if __name__ == "__main__":
    main()
