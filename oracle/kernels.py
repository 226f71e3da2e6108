"""Operator oracles: split GEMV / skinny GEMM and split paged GQA decode attention (TEST INFRASTRUCTURE).

The method reaches exactly (up to rounding order) a result with a plain definition, so each
oracle is that definition written out in float64 (SURVEY.md §8(c) "Kernel oracles"):

  * linear: C = A x B with A = weights split along M into a host
    block (leading rows [0, h)) and an HBM block (rows [h, M)); the kernel splits
    *where* rows are read from, never the arithmetic (reading R14: no split along K), so the
    result is y[n, m] = sum_k W[m, k] x[n, k] over the logical concatenation W_host (+) W_hbm.
    Optional epilogue (the decoder-layer glue of the north star): + bias[m], activation,
    + residual[n, m].
  * attention (SDPA interface over a KV cache partitioned across tiers; P:L386 decode
    attention): for request b, query head h, kv head g = floor(h * Hkv / Hq); K, V gathered by
    walking block_table[b] (bit 31 selects the host pool, low bits index the page) up to
    seq_len[b]; o = softmax(scale * K q) V with scale = 1/sqrt(d) (SDPA default).

bf16 inputs arrive as raw uint16 bits (synth module) and are decoded here by the bit-level
definition bf16 -> fp32 (bits << 16).
"""
from __future__ import annotations

import math

import numpy as np

HOST_BIT = np.uint32(0x80000000)


def bf16_to_f64(bits) -> np.ndarray:
    """Exact bf16 -> float64 decode: the bf16 pattern is the top half of an IEEE float32."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def round_to_bf16(v) -> np.ndarray:
    """Round float64 values to the nearest bf16 (ties to even), returned as float64.

    The GPU stores fp32 results as bf16 with round-to-nearest-even; for an exact (integer)
    accumulation this is the exact expected stored value. Direct f64 -> bf16 (no f32 detour):
    v = m * 2^e with m in [0.5, 1); bf16 keeps 8 significant bits -> rint(m * 2^8) / 2^8 * 2^e
    (np.rint rounds half to even). Subnormal bf16 results are out of scope (|v| >= 2^-126)."""
    v = np.asarray(v, dtype=np.float64)
    m, e = np.frexp(v)
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)


def bf16_bits_rne(v) -> np.ndarray:
    """bf16 bit patterns (uint16) of float64 values rounded to nearest even (round_to_bf16): the
    rounded values are exactly representable, so their float32 images carry them in the top half."""
    r = round_to_bf16(v).astype(np.float32)
    return (r.view(np.uint32) >> 16).astype(np.uint16)


def _act(t: np.ndarray, act: str) -> np.ndarray:
    if act == "none":
        return t
    if act == "relu":  # OPT fc1 activation
        return np.maximum(t, 0.0)
    if act == "silu":
        return t / (1.0 + np.exp(-t))
    raise ValueError(act)


def linear_rowloop(W_bits, x_bits) -> np.ndarray:
    """y[n, m] = sum_k W[m,k] x[n,k] as an explicit per-row float64 loop (C = A x B)."""
    W = bf16_to_f64(W_bits)
    x = bf16_to_f64(x_bits)
    M = W.shape[0]
    N = x.shape[0]
    y = np.zeros((N, M), dtype=np.float64)
    for m in range(M):
        row = W[m]
        for n in range(N):
            y[n, m] = float(np.dot(row, x[n]))
    return y


def linear(W_bits, x_bits, bias_bits=None, act: str = "none", residual_bits=None) -> np.ndarray:
    """Linear op with the decoder-layer epilogue, float64 (matmul as a library step, §8(c))."""
    W = bf16_to_f64(W_bits)
    x = bf16_to_f64(x_bits)
    t = x @ W.T
    if bias_bits is not None:
        t = t + bf16_to_f64(bias_bits)[None, :]
    t = _act(t, act)
    if residual_bits is not None:
        t = t + bf16_to_f64(residual_bits)
    return t


def split_linear(W_host_bits, W_hbm_bits, x_bits, **kw) -> np.ndarray:
    """Split-source linear: W is the row concatenation host (+) HBM (R7)."""
    parts = [p for p in (W_host_bits, W_hbm_bits) if p is not None and np.asarray(p).shape[0] > 0]
    W = np.concatenate([np.asarray(p, dtype=np.uint16) for p in parts], axis=0)
    return linear(W, x_bits, **kw)


def gather_kv(pool_hbm, pool_host, block_table_row, seq_len: int, g: int, page_size: int) -> np.ndarray:
    """Logical [seq_len, d] rows of one kv head, walking the block table (tier bit = bit 31)."""
    rows = []
    n_pages = -(-seq_len // page_size)
    for p in range(n_pages):
        e = np.uint32(np.int64(block_table_row[p]) & 0xFFFFFFFF)
        idx = int(e & np.uint32(0x7FFFFFFF))
        pool = pool_host if (e & HOST_BIT) else pool_hbm
        rows.append(np.asarray(pool[idx, g], dtype=np.uint16))
    K = np.concatenate(rows, axis=0)[:seq_len]
    return bf16_to_f64(K)


def paged_attention(q_bits, k_hbm, v_hbm, k_host, v_host, block_table, seq_lens, page_size: int,
                    scale: float = 0.0) -> np.ndarray:
    """Decode attention over a tier-split paged KV cache, float64.

    q_bits [B, Hq, d]; pools [P_tier, Hkv, page_size, d] (logical token-major rows);
    block_table [B, max_pages] int32 (bit 31 = host tier); seq_lens [B] (>= 1).
    Returns o [B, Hq, d] float64.
    """
    q = bf16_to_f64(q_bits)
    B, Hq, d = q.shape
    Hkv = np.asarray(k_hbm if k_hbm is not None and np.asarray(k_hbm).size else k_host).shape[1]
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0")
    grp = Hq // Hkv
    sc = scale if scale else 1.0 / math.sqrt(d)
    out = np.zeros((B, Hq, d), dtype=np.float64)
    for b in range(B):
        L = int(seq_lens[b])
        if L < 1:
            raise ValueError("seq_len must be >= 1")
        for g in range(Hkv):
            K = gather_kv(k_hbm, k_host, block_table[b], L, g, page_size)
            V = gather_kv(v_hbm, v_host, block_table[b], L, g, page_size)
            for hh in range(grp):
                h = g * grp + hh
                s = sc * (K @ q[b, h])
                s = s - s.max()
                p = np.exp(s)
                p = p / p.sum()
                out[b, h] = p @ V
    return out


def attention_dense(q_bits, K_list, V_list, scale: float = 0.0) -> np.ndarray:
    """Same definition over logical per-request K, V [L_b, Hkv, d] (no paging) — used to pin the
    paged oracle's gather against a layout-free statement of SDPA decode."""
    q = bf16_to_f64(q_bits)
    B, Hq, d = q.shape
    out = np.zeros((B, Hq, d))
    for b in range(B):
        K = bf16_to_f64(K_list[b])
        V = bf16_to_f64(V_list[b])
        Hkv = K.shape[1]
        grp = Hq // Hkv
        sc = scale if scale else 1.0 / math.sqrt(d)
        for h in range(Hq):
            g = h // grp
            s = sc * (K[:, g, :] @ q[b, h])
            p = np.exp(s - s.max())
            out[b, h] = (p / p.sum()) @ V[:, g, :]
    return out


def lse_merge(partials_o, partials_lse) -> np.ndarray:
    """Split-KV merge (flash-decoding): o = sum_c exp(lse_c - LSE) o_c, LSE = log sum_c exp(lse_c).

    Exact identity of softmax over a concatenation; used to pin split-KV chunking (float64)."""
    lse = np.asarray(partials_lse, dtype=np.float64)
    m = lse.max()
    w = np.exp(lse - m)
    w = w / w.sum()
    return np.tensordot(w, np.asarray(partials_o, dtype=np.float64), axes=(0, 0))


def rmsnorm(x, w, eps: float = 1e-5) -> np.ndarray:
    """RMSNorm over the last dim in float64 (Llama decoder layer glue, BASELINE C3 model):
    x / sqrt(mean(x^2) + eps) * w."""
    x = np.asarray(x, dtype=np.float64)
    ms = (x * x).mean(axis=-1, keepdims=True)
    return x / np.sqrt(ms + eps) * w


def layernorm(x, w, b, eps: float = 1e-5) -> np.ndarray:
    """LayerNorm over the last dim in float64 (OPT decoder layer glue)."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * w + b


def paged_prefill_attention(q_bits, k_hbm, v_hbm, k_host, v_host, block_table, seq_lens, page_size: int,
                            scale: float = 0.0) -> np.ndarray:
    """Causal prefill attention over a tier-split paged KV cache, float64 (
    P:L388 "prefill attention ... arithmetic intensity O(L)", P:L631 SDPA).

    q_bits [B, T, Hq, d]: the T newest tokens of request b, at positions L_b - T .. L_b - 1
    (L_b = seq_lens[b] >= T; their K / V rows are already in the cache). Query i attends keys
    0 .. L_b - T + i (causal); kv head g = h // (Hq / Hkv). Returns o [B, T, Hq, d] float64.
    """
    q = bf16_to_f64(q_bits)
    B, T, Hq, d = q.shape
    Hkv = np.asarray(k_hbm if k_hbm is not None and np.asarray(k_hbm).size else k_host).shape[1]
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0")
    grp = Hq // Hkv
    sc = scale if scale else 1.0 / math.sqrt(d)
    out = np.zeros((B, T, Hq, d), dtype=np.float64)
    for b in range(B):
        L = int(seq_lens[b])
        if L < T:
            raise ValueError("seq_len < T")
        for g in range(Hkv):
            K = gather_kv(k_hbm, k_host, block_table[b], L, g, page_size)
            V = gather_kv(v_hbm, v_host, block_table[b], L, g, page_size)
            for i in range(T):
                n = L - T + i + 1  # keys visible to query i
                for hh in range(grp):
                    h = g * grp + hh
                    s = sc * (K[:n] @ q[b, i, h])
                    p = np.exp(s - s.max())
                    out[b, i, h] = (p / p.sum()) @ V[:n]
    return out
