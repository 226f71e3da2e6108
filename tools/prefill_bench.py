"""Prefill attention over the tier-split KV (dak_prefill_attention): achieved
TFLOP/s and the compute-bound offload regime (an op whose compute time T exceeds its
memory time can put y <= B_h * T bytes on the host at no cost -- the planner's Phase 2).

Llama-3-70B TP8 shard shape (1 kv head x 8 q heads, d = 128), B requests of L cached tokens whose
last T are the prefill chunk; the oldest round(x * pages) pages of every request on the host.
Each host tile is read by every query block of its (request, kv head) -- T*G/128 CTAs -- so the
link carries x * KV * T*G/128 bytes (the read amplification of Table 1, for attention).
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


def run(B, L, T, Hq, Hkv, x, page=64, reps=5):
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
    dak.prefill_attention(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dak.prefill_attention(*args)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    dak.host_free(kh[0])
    dak.host_free(vh[0])
    n_keys = sum(L - T + i + 1 for i in range(T))
    flops = 4.0 * B * n_keys * Hq * d
    kv_bytes = 2 * B * L * Hkv * d * 2
    host_bytes = 2 * ht * Hkv * d * 2
    amp = -(-T * (Hq // Hkv) // 128)
    return dict(B=B, L=L, T=T, Hq=Hq, Hkv=Hkv, x=round(hp / pages, 4), us=round(t * 1e6, 1),
                tflops=round(flops / t / 1e12, 1), kv_bytes=kv_bytes, host_bytes=host_bytes, amplification=amp,
                link_gbs=round(host_bytes * amp / t / 1e9, 2))


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
    torch.cuda.set_device(0)
    base = None
    for Hq, Hkv in ((8, 1), (64, 8)):
        for x in (0.0, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5):
            r = run(B, L, T, Hq, Hkv, x)
            if x == 0.0:
                base = r["us"] * 1e-6
            # free-offload limit of the model (P:L429 with read amplification a): y <= B_h * T / a
            r["model_free_host_fraction"] = round(min(1.0, 51.5e9 * base / r["amplification"] / r["kv_bytes"]), 4)
            r["slowdown_vs_x0"] = round(r["us"] * 1e-6 / base, 3)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
