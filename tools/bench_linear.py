"""Kernel-level timing of dak_linear (development tool; bench.py is the contract harness).

Times a CUDA graph of back-to-back split linears, rotating >= 4 x L2 of distinct HBM weight
copies (and distinct host copies), and prints algorithmic GB/s per configuration as JSON lines.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

L2 = 132644864


def setup(M, K, N, h, kc, copies):
    hbm = [torch.randn((M - h) * K, device="cuda").to(torch.bfloat16).view(torch.int16) if h < M else None
           for _ in range(copies)]
    hosts = []
    for _ in range(copies if h else 0):
        hp, dp = dak.host_alloc(max(h * K * 2, 16))
        hosts.append((hp, dp))
        src = (torch.randn(h * K, device="cuda") * 0.01).to(torch.bfloat16)
        dak.pack_linear(src, h, K, kc, dp)
    x = torch.randn(N, 2 * K, device="cuda").to(torch.bfloat16)  # [gate | up] when swiglu
    y = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    return hbm, hosts, x, y


def time_cfg(M, K, N, h, kc, launches=64, reps=10, ln=False, stats=False, swiglu=False, ws=False, **cfg):
    size = M * K * 2
    copies = max(2, min(64, int(np.ceil(4 * L2 / max(size, 1)))))
    hbm, hosts, x, y = setup(M, K, N, h, kc, copies)
    lnw = torch.ones(K, device="cuda", dtype=torch.bfloat16)
    lnb = torch.zeros(K, device="cuda", dtype=torch.bfloat16)
    st_in = torch.zeros((148, N, 4), device="cuda", dtype=torch.float32)
    st_in[:, :, 0] = K / 148.0
    st_in[:, :, 2] = K / 148.0
    st_out = torch.zeros((1024, N, 4), device="cuda", dtype=torch.float32)
    ln_kw = dict(ln_w=lnw, ln_b=lnb, ln_stats=st_in, ln_parts=148) if ln else {}
    args = []
    for i in range(launches):
        a = dak.linear_args(hosts[i % copies][1] if h else None, hbm[i % copies], M, K, h, kc, N, x, y, cfg=cfg,
                            stats_out=st_out if stats else None, x_swiglu=int(swiglu), **ln_kw)
        args.append(a)
    wsb = None
    if ws:
        need = dak.linear_workspace_size(args[0])
        if need:
            wsb = torch.zeros(need, dtype=torch.uint8, device="cuda")
            for a in args:
                a.workspace, a.workspace_bytes = wsb.data_ptr(), need
    info = dak.linear_query(args[0])
    info["ws"] = dak.linear_workspace_size(args[0]) if ws else 0
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for a in args[:4]:
            dak.linear(a, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for a in args:
                dak.linear(a, s)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / launches * 1e-3)
    t = float(np.median(ts))
    alg = size + N * K * 2 + N * M * 2
    for hp, _ in hosts:
        dak.host_free(hp)
    del hbm
    torch.cuda.empty_cache()
    return dict(M=M, K=K, N=N, h=h, kc=kc, ln=ln, stats=stats, swiglu=swiglu, us=t * 1e6, gbs=alg / t / 1e9, hbm_gbs=(M - h) * K * 2 / t / 1e9,
                host_gbs=h * K * 2 / t / 1e9, info={k: info[k] for k in ("grid", "n_cta_host", "stages_hbm", "window_host",
                                                                        "smem_bytes", "path", "ws")}, cfg=cfg)


def time_chain(layers=8, N=8, two_per_sm=False, stages=0, kc_override=0):
    """OPT-30B layer linears (qkv, o, fc1, fc2) x layers chained with PDL in one graph, host share r*;
    two_per_sm: two CTAs per SM per op (rows halved, ring <= 113 KB) so the next op's CTAs can take
    a slot while this op's last CTAs drain."""
    H, F = 7168, 28672
    shapes = [(3 * H, H), (H, H), (F, H), (H, F)] * layers
    sms = dak.device_sms()
    args, keep = [], []
    x = torch.randn(N, F, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, F, device="cuda", dtype=torch.bfloat16)
    for (M, K) in shapes:
        h = 16 * max(1, round(M * 0.0066 / 16))
        nh = 2
        nhbm = (2 * sms - nh) if two_per_sm else 0
        rows = -(-(M - h) // (nhbm or (sms - nh)))
        kc = kc_override or dak.choose_kc(rows, K)
        W = torch.randn((M - h) * K, device="cuda").to(torch.bfloat16)
        hp, dp = dak.host_alloc(h * K * 2)
        keep += [W, hp]
        cfg = dict(pdl=1, congestion_control=1, n_cta_host=nh, n_cta_hbm=nhbm, stages=stages)
        args.append(dak.linear_args(dp, W, M, K, h, kc, N, x, y, cfg=cfg))
    info = [dak.linear_query(a) for a in args[:4]]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for a in args:
            dak.linear(a, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for a in args:
                dak.linear(a, s)
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
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(ts))
    nbytes = sum(M * K * 2 for M, K in shapes)
    for hp in keep[1::2]:
        dak.host_free(hp)
    return dict(two_per_sm=two_per_sm, stages=stages, ms=round(t * 1e3, 4), gbs=round(nbytes / t / 1e9, 1),
                info=[{k: i[k] for k in ("grid", "smem_bytes", "stages_hbm")} for i in info])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--exp", default="")
    a = ap.parse_args()
    if a.exp == "chain":  # OPT layer chain: one CTA per SM (default) vs two per SM with shallower rings
        print(json.dumps(time_chain()), flush=True)
        for st in (2, 3, 4):
            try:
                print(json.dumps(time_chain(two_per_sm=True, stages=st)), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(two_per_sm=True, stages=st, error=str(e))), flush=True)
        return
    if a.exp == "n16":  # OPT-30B shapes at N = 16: mma.sync (path 2) vs tcgen05 (3, split-K when few rows) vs swapped (4)
        for (M, K) in ((21504, 7168), (7168, 7168), (28672, 7168), (7168, 28672)):
            h = 16 * max(1, round(M * 0.0066 / 16))
            for path in (2, 3, 4):
                kc = 64 if path >= 3 else dak.choose_kc(-(-(M - h) // 146), K)
                try:
                    r = time_cfg(M, K, 16, h, kc, pdl=1, n_cta_host=2, congestion_control=1, force_path=path, ws=True)
                except Exception as e:  # noqa: BLE001
                    r = dict(M=M, K=K, path=path, error=str(e))
                print(json.dumps(r), flush=True)
        return
    if a.exp == "sk":  # tcgen05 split-K at the Llama TP8 shard shapes, b64 (kc from env KCS, default 64)
        for (M, K) in ((1280, 8192), (8192, 1024), (7168, 8192), (8192, 3584)):
            for kc in [int(v) for v in os.environ.get("KCS", "64").split(",")]:
                try:
                    r = time_cfg(M, K, 64, 0, kc, pdl=1, force_path=3, ws=True)
                except Exception as e:  # noqa: BLE001
                    r = dict(M=M, K=K, kc=kc, error=str(e))
                print(json.dumps(r), flush=True)
        return
    if a.exp == "tcx":  # tcgen05 operand transforms at the Llama TP8 shard shapes, b64
        for (M, K, kw) in ((8192, 3584, dict(swiglu=True)), (7168, 8192, dict(ln=True)), (8192, 3584, {}),
                           (7168, 8192, {})):
            for path in (2, 3):
                kc = 64 if path == 3 else 256
                try:
                    r = time_cfg(M, K, 64, 0, kc, pdl=1, force_path=path, **kw)
                    print(json.dumps(r), flush=True)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps(dict(M=M, K=K, path=path, error=str(e))), flush=True)
        return
    if a.exp == "tc":  # tcgen05 (path 3, kc 64) vs mma.sync (path 2) at growing N
        for (M, K) in ((7168, 8192), (28672, 7168), (1024, 8192)):
            for N in (8, 16, 32, 64, 128, 256):
                for path in ((2, 3) if N <= 64 else (3,)):
                    kc = 64 if path == 3 else dak.default_kc(M, K, 147)
                    try:
                        r = time_cfg(M, K, N, 0, kc, pdl=1, force_path=path)
                        print(json.dumps(r), flush=True)
                    except Exception as e:  # noqa: BLE001
                        print(json.dumps(dict(M=M, K=K, N=N, path=path, error=str(e))), flush=True)
        return
    if a.exp == "mc":  # x multicast within clusters (one fetch per cluster)
        for (M, K, h, kc, N) in ((7168, 7168, 48, 256, 8), (28672, 7168, 192, 64, 8), (7168, 8192, 48, 256, 64),
                                 (1024, 8192, 16, 256, 64)):
            for cl in (1, 2, 4):
                print(json.dumps(time_cfg(M, K, N, h, kc, pdl=1, n_cta_host=2, congestion_control=1, cluster=cl)),
                      flush=True)
        return
    if a.exp == "ln":  # fused pre-norm / stats epilogue cost at the OPT-30B shapes (N = 8)
        for (M, K, h, kc) in ((7168, 7168, 48, 256), (28672, 7168, 192, 64)):
            for pdl in (0, 1):
                for ln, st in ((False, False), (True, False), (False, True)):
                    print(json.dumps(time_cfg(M, K, 8, h, kc, ln=ln, stats=st, pdl=pdl, n_cta_host=2,
                                              congestion_control=1)), flush=True)
        return
    shapes = [(4096, 4096), (7168, 7168), (28672, 7168), (7168, 28672)]
    Ns = [1, 8] if a.quick else [1, 2, 4, 8, 16]
    for (M, K) in shapes:
        kc = dak.default_kc(M, K, 147)
        for N in Ns:
            for h in (0, 16 * max(1, round(M * 0.0069 / 16))):
                r = time_cfg(M, K, N, h, kc)
                print(json.dumps(r), flush=True)
    # pdl on / off and stage sweep at C1
    for pdl in (0, 1):
        print(json.dumps(time_cfg(4096, 4096, 1, 32, 512, pdl=pdl)), flush=True)
    for st in (2, 3, 4, 6):
        print(json.dumps(time_cfg(28672, 7168, 8, 0, 64, stages=st)), flush=True)


if __name__ == "__main__":
    main()
