"""Link-traffic evidence for the split kernels (PAPER Table 1).

Runs each case ONCE (one profiled launch of the split kernel, after the packing kernels) so that
`ncu --metrics pcie__read_bytes.sum,syslts__t_sectors_aperture_sysmem.sum,dram__bytes_read.sum,...
-k regex:"split_linear|umma|split_attention"` captures exactly one launch per case, in the order
printed here. tools/summarize_link.py then divides the measured link bytes by each case's
algorithmic host bytes: 1x means every host byte crossed the link once (direct access, multicast);
Table 1's read amplification shows up as xG without the weight-tile multicast.

  python tools/link_counters.py > gpurun_out/link_cases.jsonl
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402


def linear_case(name, M, K, N, h, kc, **cfg):
    g = torch.Generator(device="cuda")
    g.manual_seed(M + N + h)
    W = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    hbm = torch.empty((M - h) * K, dtype=torch.bfloat16, device="cuda") if h < M else None
    host = dak.host_alloc(max(h * K * 2, 16)) if h > 0 else None
    if hbm is not None:
        dak.pack_linear(W[h:].contiguous(), M - h, K, kc, hbm)
    if host:
        dak.pack_linear(W[:h].contiguous(), h, K, kc, host[1])
    x = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, M, dtype=torch.bfloat16, device="cuda")
    a = dak.linear_args(host[1] if host else None, hbm, M, K, h, kc, N, x, y, cfg=cfg)
    a.workspace, a.workspace_bytes = 256, 1 << 40
    need = dak.linear_workspace_size(a)
    a.workspace, a.workspace_bytes = None, 0
    ws = None
    if need:
        ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
        a.workspace, a.workspace_bytes = ws.data_ptr(), need
    info = dak.linear_query(a)
    torch.cuda.synchronize()
    dak.linear(a)
    torch.cuda.synchronize()
    print(json.dumps(dict(case=name, kernel="linear", M=M, K=K, N=N, h=h, host_bytes=h * K * 2, hbm_bytes=(M - h) * K * 2,
                          x_bytes=N * K * 2, grid=info["grid"], cluster=cfg.get("cluster", 0),
                          groups=-(-N // 512) if N > 512 else 1)), flush=True)
    if host:
        dak.host_free(host[0])


def attention_case(name, B, L, Hq, Hkv, frac, page=64, cp=16):
    d = 128
    pages = -(-L // page)
    n_chunks = -(-pages // cp)
    hu_per_req = int(round(frac * n_chunks))
    bt, Ph, Pg, ht = dak.kv_place([L] * B, page, pages, cp, hu_per_req * B)
    pe = Hkv * page * d
    kg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
    vg = torch.randn_like(kg)
    kh, vh = dak.host_alloc(max(Ph, 1) * pe * 2), dak.host_alloc(max(Ph, 1) * pe * 2)
    q = torch.randn(B, Hq, d, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    btd = torch.from_numpy(bt).cuda()
    a = dak.attention_args(q, out, kg, vg, kh[1], vh[1], btd, sl, B, Hq, Hkv, d, page, pages, cp,
                           cfg=dict(pdl=1, congestion_control=1, n_cta_host=0))
    ws = torch.zeros(max(dak.attention_workspace_size(a), 16), dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    torch.cuda.synchronize()
    dak.attention(a)
    torch.cuda.synchronize()
    tok = 2 * Hkv * d * 2
    print(json.dumps(dict(case=name, kernel="attention", B=B, L=L, Hq=Hq, Hkv=Hkv, host_bytes=ht * tok,
                          hbm_bytes=(B * L - ht) * tok)), flush=True)
    dak.host_free(kh[0])
    dak.host_free(vh[0])


def main():
    torch.cuda.set_device(0)
    M, K = 28672, 7168
    rs = 51.5 / (6542.1 + 51.5)
    h_star = int(round(rs * M / 16)) * 16
    linear_case("fc1_N8_rstar", M, K, 8, h_star, 64, pdl=0, congestion_control=1)
    linear_case("fc1_N8_r0.5", M, K, 8, M // 2, 64, pdl=0, congestion_control=1)
    attention_case("c4_B1_128k_r0.5", 1, 131072, 64, 8, 0.5)
    for N, r in ((1024, 0.5), (2048, 0.25)):
        h = int(round(r * 7168 / 128)) * 128
        linear_case(f"t1_N{N}_r{r}_multicast", 7168, 7168, N, h, 64, pdl=0, cluster=2)
        linear_case(f"t1_N{N}_r{r}_no_multicast", 7168, 7168, N, h, 64, pdl=0, cluster=0)


if __name__ == "__main__":
    main()
