"""Test-side helpers for GPU parity tests (test infrastructure; not product code)."""
from __future__ import annotations

import ctypes

import numpy as np


def to_dev(bits: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda()


def from_dev(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


class HostBuf:
    """Pinned + mapped host block allocated through the library (dak_host_alloc)."""

    def __init__(self, D, nbytes: int, wc: bool = False):
        self.D = D
        self.nbytes = max(int(nbytes), 16)
        self.hp, self.dp = D.host_alloc(self.nbytes, write_combined=wc)

    def numpy(self, dtype=np.uint16):
        arr = (ctypes.c_uint8 * self.nbytes).from_address(self.hp)
        return np.frombuffer(arr, dtype=np.uint8).view(dtype)

    def free(self):
        if self.hp:
            self.D.host_free(self.hp)
            self.hp = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class SplitLinear:
    """Weights W [M,K] split at row h: rows [0,h) packed into pinned host memory, rows [h,M)
    packed into HBM, both in the library's DAK-KC layout (dak_pack_linear)."""

    def __init__(self, D, W_bits: np.ndarray, h: int, kc: int):
        import torch
        self.D = D
        M, K = W_bits.shape
        self.M, self.K, self.h, self.kc = M, K, h, kc
        Wd = to_dev(W_bits)
        self.hbm = None
        self.host = None
        if h < M:
            self.hbm = torch.empty((M - h) * K, dtype=torch.int16, device="cuda")
            D.pack_linear(Wd[h:].contiguous(), M - h, K, kc, self.hbm)
        if h > 0:
            self.host = HostBuf(D, h * K * 2)
            D.pack_linear(Wd[:h].contiguous(), h, K, kc, self.host.dp)
        torch.cuda.synchronize()

    def args(self, x, y, N, bias=None, residual=None, act=0, **cfg):
        return self.D.linear_args(self.host.dp if self.host else None, self.hbm, self.M, self.K, self.h, self.kc, N,
                                  x, y, bias=bias, residual=residual, act=act, cfg=cfg)


def assert_close(got: np.ndarray, ref: np.ndarray, rtol: float = 1e-2):
    """North-star tolerance: per element |g - o| <= rtol * max(|o|, rms(o)); relative Frobenius <= rtol."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.all(np.isfinite(got)), "non-finite output"
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    err = np.abs(got - ref)
    bound = rtol * np.maximum(np.abs(ref), rms)
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(f"{bad.sum()} / {bad.size} elements out of tolerance; worst at {i}: got {got[i]} ref {ref[i]}")
    fro = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    assert fro <= rtol, fro


def make_paged_kv(Ls, Hkv, d, page, host_chunks_frac, chunk_pages, seed, Hq, kind="normal", paper_mode=False):
    """Logical KV (synth) -> logical page pools + block table. Host = the oldest
    round_half_up(frac * n_chunks) chunks of each request (DESIGN reading), or whole requests
    (paper mode). Returns q, K list, V list, (kg, vg, kh, vh, bt) with logical pools."""
    from oracle.partition import host_pages_prefix, batch_split_host_requests
    q, K, V = __import__("synth").kv_inputs(Ls, Hkv, d, Hq, seed, kind=kind)
    g = np.random.default_rng(seed + 1)
    B = len(Ls)
    pages = [-(-L // page) for L in Ls]
    max_pages = max(pages)
    if paper_mode:
        nreq = batch_split_host_requests(B, host_chunks_frac)
        n_host = [pages[b] if b < nreq else 0 for b in range(B)]
    else:
        n_host = [host_pages_prefix(pages[b], host_chunks_frac, chunk_pages) for b in range(B)]
    Ph, Pg = sum(n_host), sum(p - h for p, h in zip(pages, n_host))
    kh = np.zeros((max(Ph, 1), Hkv, page, d), np.uint16)
    vh = np.zeros_like(kh)
    kg = np.zeros((max(Pg, 1), Hkv, page, d), np.uint16)
    vg = np.zeros_like(kg)
    bt = np.zeros((B, max_pages), np.int64)
    ih = list(g.permutation(max(Ph, 1)))
    ig = list(g.permutation(max(Pg, 1)))
    for b, L in enumerate(Ls):
        for pi in range(pages[b]):
            lo, hi = pi * page, min(L, (pi + 1) * page)
            if pi < n_host[b]:
                j = int(ih.pop())
                kh[j, :, :hi - lo] = K[b][lo:hi].transpose(1, 0, 2)
                vh[j, :, :hi - lo] = V[b][lo:hi].transpose(1, 0, 2)
                bt[b, pi] = j | 0x80000000
            else:
                j = int(ig.pop())
                kg[j, :, :hi - lo] = K[b][lo:hi].transpose(1, 0, 2)
                vg[j, :, :hi - lo] = V[b][lo:hi].transpose(1, 0, 2)
                bt[b, pi] = j
    bt = (bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    return q, K, V, (kg, vg, kh, vh, bt), n_host


class PagedKV:
    """Device-side tier pools in the DAK-PG layout (packed by dak_pack_kv_pages)."""

    def __init__(self, D, kg, vg, kh, vh, bt, page, has_host=True):
        import torch
        self.D = D
        P, Hkv, pg, d = kg.shape
        self.kg = torch.empty(kg.size, dtype=torch.int16, device="cuda")
        self.vg = torch.empty(vg.size, dtype=torch.int16, device="cuda")
        D.pack_kv_pages(to_dev(kg), kg.shape[0] * Hkv, page, d, self.kg)
        D.pack_kv_pages(to_dev(vg), vg.shape[0] * Hkv, page, d, self.vg)
        self.kh = HostBuf(D, kh.size * 2)
        self.vh = HostBuf(D, vh.size * 2)
        D.pack_kv_pages(to_dev(kh), kh.shape[0] * Hkv, page, d, self.kh.dp)
        D.pack_kv_pages(to_dev(vh), vh.shape[0] * Hkv, page, d, self.vh.dp)
        self.bt = torch.from_numpy(bt.copy()).cuda()
        self.page = page
        torch.cuda.synchronize()


def assert_bf16_ulps(got: np.ndarray, ref: np.ndarray, ulps: int = 1, floor: float = 0.0):
    """Per element: |g - r| <= ulps * ulp_bf16(r) (+ floor). ref is the float64 oracle value already
    rounded to bf16; a kernel computing in fp32 may land one bf16 ulp away at a rounding boundary."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape and np.all(np.isfinite(got))
    mag = np.maximum(np.abs(ref), 2.0 ** -126)
    ulp = 2.0 ** (np.floor(np.log2(mag)) - 7)
    err = np.abs(got - ref)
    bad = err > ulps * ulp + floor
    if bad.any():
        i = np.unravel_index(np.argmax(err - ulps * ulp), err.shape)
        raise AssertionError(f"{bad.sum()} / {bad.size} elements beyond {ulps} bf16 ulp; worst at {i}: got {got[i]} ref {ref[i]}")
