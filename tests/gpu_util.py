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
