"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no dot products, no softmax, no planning):
it only draws random numbers and rounds them to the storage type (bf16, RNE), so that the
oracle (``oracle/``) and the CUDA path (``paper_2604_26074_b200``) consume identical bits.

Recipe (SURVEY.md §8(d) "Concrete synthetic inputs"):
  * generator: ``numpy.random.default_rng(seed)`` with ``seed = 0xDA0 + config_index + 1000*op_index``;
  * floating values are drawn in float32 then rounded to bf16 with round-to-nearest-even;
  * linear weights ~ N(0, 1/K), activations ~ N(0, 1), KV ~ N(0, 1), queries ~ N(0, 1);
  * the "int" variant draws integers in [-2, 2] (exactly representable in bf16), used for
    bit-exact parity (all partial sums are small integers, exact in fp32 in any order).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0xDA0


def seed_for(config_index: int, op_index: int = 0) -> int:
    """Seed convention of SURVEY.md §8(d): 0xDA0 + config index + 1000 * op index."""
    return SEED_BASE + int(config_index) + 1000 * int(op_index)


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(int(seed))


def bf16_bits(a) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even) and return the raw uint16 bits.

    NaN is not produced by any generator here; +-Inf cannot arise from the bounded draws.
    """
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = (u + 0x7FFF + lsb) >> 16
    return r.astype(np.uint16)


def normal_bf16(g: np.random.Generator, shape, std: float = 1.0) -> np.ndarray:
    return bf16_bits(g.standard_normal(size=shape, dtype=np.float32) * np.float32(std))


def int_bf16(g: np.random.Generator, shape, lo: int = -2, hi: int = 2) -> np.ndarray:
    return bf16_bits(g.integers(lo, hi + 1, size=shape).astype(np.float32))


def linear_inputs(M: int, K: int, N: int, seed: int, kind: str = "normal", bias: bool = False):
    """Weights W [M,K], activations x [N,K] (and optional bias [M]) as bf16 bits."""
    g = rng(seed)
    if kind == "normal":
        W = normal_bf16(g, (M, K), std=1.0 / np.sqrt(K))
        x = normal_bf16(g, (N, K))
        b = normal_bf16(g, (M,), std=0.1) if bias else None
    elif kind == "int":
        W = int_bf16(g, (M, K))
        x = int_bf16(g, (N, K))
        b = int_bf16(g, (M,)) if bias else None
    else:
        raise ValueError(kind)
    return W, x, b


def kv_inputs(n_tokens_per_req, Hkv: int, d: int, Hq: int, seed: int, kind: str = "normal"):
    """Logical per-request K, V [L_b, Hkv, d] and queries q [B, Hq, d] as bf16 bits."""
    g = rng(seed)
    B = len(n_tokens_per_req)
    draw = int_bf16 if kind == "int" else normal_bf16
    # score-range variants (parity of the online softmax's rescaling and the combine's max
    # tracking): "wide" draws q with std 40 (scores ~ N(0, 40^2) after the 1/sqrt(d) scale);
    # "constk" repeats one key row over every token (softmax uniform: o = mean V); "dominant"
    # puts a key of +-3 signs matching q's first head at a random token of every request, with q
    # std 4 (that key's score exceeds the others by ~100)
    q = draw(g, (B, Hq, d)) if kind == "int" else normal_bf16(
        g, (B, Hq, d), 40.0 if kind == "wide" else (4.0 if kind == "dominant" else 1.0))
    K = [draw(g, (int(L), Hkv, d)) for L in n_tokens_per_req]
    V = [draw(g, (int(L), Hkv, d)) for L in n_tokens_per_req]
    if kind == "constk":
        K = [np.repeat(k[:1], k.shape[0], axis=0) for k in K]
    elif kind == "dominant":
        qf = (q.astype(np.uint32) << 16).view(np.float32)
        for b, k in enumerate(K):
            t = int(g.integers(0, k.shape[0]))
            for j in range(Hkv):
                k[t, j] = bf16_bits(np.where(qf[b, j * (Hq // Hkv)] >= 0, 3.0, -3.0).astype(np.float32))
    return q, K, V


def random_ops(g: np.random.Generator, n_ops: int, units_max: int = 8):
    """Random planner op lists for brute-force pins: (n_units, unit_bytes, T_seconds) tuples.

    unit bytes are drawn in GB-scale integers so that exact Fraction arithmetic stays small.
    """
    ops = []
    for _ in range(n_ops):
        n = int(g.integers(1, units_max + 1))
        u = int(g.integers(1, 50)) * 10**8
        ops.append((n, u))
    return ops
