"""Prefill attention over the tier-split KV (dak_prefill_attention): achieved
TFLOP/s and the compute-bound offload regime (an op whose compute time T exceeds its
memory time can put y <= B_h * T bytes on the host at no cost -- the planner's Phase 2).

Llama-3-70B TP8 shard shape (1 kv head x 8 q heads, d = 128), B requests of L cached tokens whose
last T are the prefill chunk; the oldest round(x * pages) pages of every request on the host.
With the staging workspace, 4 streamer CTAs read every host page once over the link while the
compute CTAs work newest keys first (amplification 1); without it every query block of a
(request, kv head) -- T*G/128 CTAs -- reads the host tiles itself (Table 1's read amplification,
P:L537-558, for attention).
Prints one JSON line per point: time, TFLOP/s (causal FLOPs 4 * sum_i n_i * Hq * d), link GB/s,
and the model's free-offload limit y_free = B_h * t(x=0) / amplification.

  python tools/prefill_bench.py [B] [L] [T]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402


def run(B, L, T, Hq, Hkv, x, page=64, reps=5, stage=True):
    d = 128
    pages = -(-L // page)
    hp = int(round(x * pages))
    bt, Ph, Pg, ht = dak.kv_place([L] * B, page, pages, 1, hp * B)  # chunk = 1 page: per-request prefix
    pe = Hkv * page * d
    kg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
    vg = torch.randn_like(kg)
    kh, vh = dak.host_alloc(max(Ph, 1) * pe * 2), dak.host_alloc(max(Ph, 1) * pe * 2)
    q = torch.randn(B, T, Hq, d, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    btd = torch.from_numpy(bt).cuda()
    args = (q, out, kg, vg, kh[1], vh[1], btd, sl, B, T, Hq, Hkv, d, page, pages)
    ws = torch.empty(dak.prefill_workspace_size(B, Hkv, page, pages), dtype=torch.uint8, device="cuda") if stage else None
    kw = dict(workspace=ws, workspace_bytes=ws.numel() if ws is not None else 0)
    dak.prefill_attention(*args, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dak.prefill_attention(*args, **kw)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    dak.host_free(kh[0])
    dak.host_free(vh[0])
    n_keys = sum(L - T + i + 1 for i in range(T))
    flops = 4.0 * B * n_keys * Hq * d
    kv_bytes = 2 * B * L * Hkv * d * 2
    host_bytes = 2 * ht * Hkv * d * 2
    amp = 1 if stage else -(-T * (Hq // Hkv) // 128)  # streamed once, or once per query block
    return dict(B=B, L=L, T=T, Hq=Hq, Hkv=Hkv, x=round(hp / pages, 4), staged=stage, us=round(t * 1e6, 1),
                tflops=round(flops / t / 1e12, 1), kv_bytes=kv_bytes, host_bytes=host_bytes, amplification=amp,
                link_gbs=round(host_bytes * amp / t / 1e9, 2))


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
    torch.cuda.set_device(0)
    base = None
    for Hq, Hkv, stage in ((8, 1, True), (64, 8, True), (8, 1, False)):
        for x in ((0.0, 0.02, 0.05, 0.1, 0.2, 0.3, 0.5, 0.75, 1.0) if stage else (0.0, 0.01, 0.05, 0.2)):
            r = run(B, L, T, Hq, Hkv, x, stage=stage)
            if x == 0.0:
                base = r["us"] * 1e-6
            # free-offload limit of the model (P:L429 with read amplification a): y <= B_h * T / a
            r["model_free_host_fraction"] = round(min(1.0, 51.5e9 * base / r["amplification"] / r["kv_bytes"]), 4)
            r["slowdown_vs_x0"] = round(r["us"] * 1e-6 / base, 3)
            if stage:  # the planner on this op (T_comp = the measured all-HBM time): its phase and latency
                page_kv = 2 * Hkv * 64 * 128 * 2
                op = dict(kind="attention", n_units=B * (L // 64), unit_bytes=page_kv, total_bytes=r["kv_bytes"], T=base)
                pl, _ = dak.plan_ratios(dict(hbm_bps=6542.1e9, link_bps=51.5e9), [op], r["host_bytes"], dak.PLAN_EXACT)
                r["planner_phase"], r["planner_latency_us"] = pl[0]["phase"], round(pl[0]["latency"] * 1e6, 1)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
