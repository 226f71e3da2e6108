"""Measurement sweeps for BASELINE configs C1, C4, C5 (development tool; bench.py is the contract):

  c5   fc1 28672x7168 at N=8 (and the C1 GEMV 4096^2 at N=1) over the host ratio r, congestion
       control on/off: achieved (HBM + link) GB/s vs the split roofline
       EB(r) = 1 / max((1 - r) / B_g, r / B_l)  (equals B_g + B_l at r* = B_l / (B_g + B_l))
  c4   GQA decode attention, 64 q / 8 kv heads, 131072 tokens, B in {1, 4}, host share r of the
       oldest KV chunks in {0, r*, 0.5}
  pf   direct split access vs the prefetch-to-HBM baseline (copy the host rows into HBM
       with the copy engine, then run the GEMV from HBM) on fc1 28672x7168 at N=8 over r
  t1   Table 1 on B200: the 7168 x 7168 matrix at N in {256 .. 4096}, host share r;
       N > 512 runs as groups of N/512 CTAs with and without the weight-tile multicast (without it
       every host tile crosses the link N/512 times: Table 1's read amplification)
Prints one JSON line per point. B_g: MEASURED_PEAKS.json HBM copy; B_l: measured link 51.5 GB/s.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402
from tools.bench_linear import time_cfg  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks():
    bg = 6555.5e9
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_bw_gbs"):
            if k in d:
                bg = float(d[k]) * 1e9
                break
    return bg, 51.5e9


def eb(r, bg, bl):
    return 1.0 / max((1 - r) / bg, r / bl if r > 0 else 0.0)


def c5():
    bg, bl = peaks()
    rs = bl / (bg + bl)
    for (M, K, N, kc) in ((28672, 7168, 8, 64), (4096, 4096, 1, 512)):
        unit = 16
        for r in sorted({0.0, rs / 2, rs, 2 * rs, 0.02, 0.05, 0.1, 0.2, 0.3, 0.5, 0.7, 1.0}):
            h = min(M, int(round(r * M / unit)) * unit)
            for cc in (1, 0):
                if h == 0 and cc == 0:
                    continue
                res = time_cfg(M, K, N, h, kc, launches=16 if h > M // 4 else 64, reps=5, pdl=1, n_cta_host=0,
                               congestion_control=cc)
                rr = h / M
                print(json.dumps(dict(exp="c5", M=M, K=K, N=N, r=round(rr, 5), h=h, cc=cc, us=round(res["us"], 2),
                                      gbs=round(res["hbm_gbs"] + res["host_gbs"], 1), host_gbs=round(res["host_gbs"], 2),
                                      roofline_gbs=round(eb(rr, bg, bl) / 1e9, 1),
                                      frac=round((res["hbm_gbs"] + res["host_gbs"]) * 1e9 / eb(rr, bg, bl), 4),
                                      n_cta_host=res["info"]["n_cta_host"], window=res["info"]["window_host"])),
                      flush=True)


def c4():
    bg, bl = peaks()
    rs = bl / (bg + bl)
    d, Hq, Hkv, L, page = 128, 64, 8, 131072, 64
    cp = int(os.environ.get("DAK_C4_CHUNK_PAGES", "16"))
    for B in (1, 4):
        pages = L // page
        for r in (0.0, rs, 0.5):
            n_chunks = pages // cp
            host_chunks = int(round(r * n_chunks))
            hp = host_chunks * cp  # oldest pages of each request on the host
            Ph, Pg = B * hp, B * (pages - hp)
            pe = Hkv * page * d
            kg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
            vg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
            kh = dak.host_alloc(max(Ph, 1) * pe * 2)
            vh = dak.host_alloc(max(Ph, 1) * pe * 2)
            bt = np.zeros((B, pages), np.int64)
            ih = ig = 0
            for b in range(B):
                for pgi in range(pages):
                    if pgi < hp:
                        bt[b, pgi] = ih | 0x80000000
                        ih += 1
                    else:
                        bt[b, pgi] = ig
                        ig += 1
            btd = torch.from_numpy((bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda()
            q = torch.randn(B, Hq, d, device="cuda").to(torch.bfloat16)
            out = torch.empty_like(q)
            sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
            for cc in ((1, 0) if hp else (1,)):
                nh = 0  # auto: the library picks the host CTAs from the block table
                a = dak.attention_args(q, out, kg, vg, kh[1], vh[1], btd, sl, B, Hq, Hkv, d, page, pages, cp,
                                       cfg=dict(pdl=1, congestion_control=cc, n_cta_host=nh))
                ws = torch.zeros(dak.attention_workspace_size(a), dtype=torch.uint8, device="cuda")
                a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    dak.attention(a, s)
                    s.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        for _ in range(4):
                            dak.attention(a, s)
                torch.cuda.synchronize()
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ts = []
                for _ in range(5):
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 4 * 1e-3)
                t = float(np.median(ts))
                kv = 2 * B * L * Hkv * d * 2
                rr = hp / pages
                print(json.dumps(dict(exp="c4", B=B, L=L, Hq=Hq, Hkv=Hkv, r=round(rr, 5), cc=cc, us=round(t * 1e6, 1),
                                      gbs=round(kv / t / 1e9, 1), roofline_gbs=round(eb(rr, bg, bl) / 1e9, 1),
                                      frac=round(kv / t / eb(rr, bg, bl), 4))), flush=True)
            dak.host_free(kh[0])
            dak.host_free(vh[0])
            del kg, vg
            torch.cuda.empty_cache()


def _cudart():
    import ctypes
    import glob
    for cand in glob.glob("/usr/local/cuda/lib64/libcudart.so*") + ["libcudart.so.12", "libcudart.so"]:
        try:
            lib = ctypes.CDLL(cand)
            lib.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                            ctypes.c_void_p]
            return lib
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def pf():
    """Per r: (a) direct: one dak_linear reading the h host rows over the link while the rest
    streams from HBM (DAK); (b) prefetch: cudaMemcpyAsync (copy engine) of the h host rows into
    HBM, then one all-HBM dak_linear. Both timed per call with events, median of 5."""
    bg, bl = peaks()
    M, K, N, kc = 28672, 7168, 8, 64
    rs = bl / (bg + bl)
    rt = _cudart()
    x = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    w_all = torch.randn(M * K, device="cuda").to(torch.bfloat16)  # HBM image of the whole matrix
    for r in sorted({0.0, rs, 2 * rs, 0.02, 0.05, 0.1, 0.2, 0.5}):
        h = min(M, int(round(r * M / 16)) * 16)
        hp, dp = dak.host_alloc(max(h * K * 2, 16))
        if h:
            dak.pack_linear(torch.randn(h * K, device="cuda").to(torch.bfloat16), h, K, kc, dp)
        direct = dak.linear_args(dp if h else None, w_all[h * K:], M, K, h, kc, N, x, y, cfg=dict(pdl=0))
        pref = dak.linear_args(None, w_all, M, K, 0, kc, N, x, y, cfg=dict(pdl=0))
        s_ = torch.cuda.Stream()
        times = {}
        for name in ("direct", "prefetch"):
            def run():
                if name == "direct":
                    dak.linear(direct, s_)
                else:
                    if h:
                        assert rt.cudaMemcpyAsync(w_all.data_ptr(), hp, h * K * 2, 1, s_.cuda_stream) == 0
                    dak.linear(pref, s_)
            run()
            s_.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(5):
                e0.record(s_)
                run()
                e1.record(s_)
                s_.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            times[name] = float(np.median(ts))
        print(json.dumps(dict(exp="pf", M=M, K=K, N=N, r=round(h / M, 5), h=h, direct_us=round(times["direct"], 1),
                              prefetch_us=round(times["prefetch"], 1),
                              speedup_direct_over_prefetch=round(times["prefetch"] / times["direct"], 3))), flush=True)
        dak.host_free(hp)


def t1():
    bg, bl = peaks()
    M = K = 7168
    for N in (256, 512, 1024, 2048, 4096):
        for r in ((0.0, 0.25, 0.5) if N <= 1024 else (0.25,)):
            h = int(round(r * M / 128)) * 128
            for cl in ((0, 2) if N > 512 else (0,)):
                res = time_cfg(M, K, N, h, 64, launches=8 if h else 32, reps=3, pdl=1, cluster=cl, ws=True)
                t = res["us"] * 1e-6
                amp = -(-N // 512) if (N > 512 and cl != 2) else 1  # host fetches of a tile per CTA group
                rr = h / M
                print(json.dumps(dict(exp="t1", M=M, K=K, N=N, r=round(rr, 4), multicast=int(cl == 2) if N > 512 else None,
                                      us=round(res["us"], 1), alg_gbs=round(res["hbm_gbs"] + res["host_gbs"], 1),
                                      link_bytes_moved=h * K * 2 * amp, link_gbs_moved=round(h * K * 2 * amp / t / 1e9, 2),
                                      tflops=round(2.0 * M * N * K / t / 1e12, 1),
                                      roofline_gbs=round(eb(rr, bg, bl) / 1e9, 1),
                                      frac=round((res["hbm_gbs"] + res["host_gbs"]) * 1e9 / eb(rr, bg, bl), 4),
                                      grid=res["info"]["grid"])), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c5", "c4"]
    for w in which:
        globals()[w]()
