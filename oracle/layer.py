"""Decoder-layer / decode-step oracle for the OPT family (TEST INFRASTRUCTURE).

The paper integrates its split kernels as drop-in replacements of nn.Linear and SDPA inside the
model and evaluates OPT models decoding one token per step; the offloaded
operators compute exactly what the un-offloaded model computes. This oracle is therefore the
plain OPT decoder decode step (pre-LayerNorm, biases, ReLU MLP, learned positions with offset 2,
tied LM head), in float64 with no intermediate rounding:

    h = LN1(x); [q k v] = h Wqkv^T + b; K,V += k,v; a = SDPA(q, K, V); x = x + a Wo^T + bo
    h = LN2(x); x = x + relu(h W1^T + b1) W2^T + b2
    logits = LN_f(x) E^T

Parameters are bf16 bit arrays (synth module); KV caches are logical per-request arrays.
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import bf16_to_f64, layernorm


def opt_decode_layer(x, p: dict, K_prev: list, V_prev: list, n_heads: int, eps: float = 1e-5):
    """One layer. x: float64 [B, H]; p: bf16-bit params (qkv [3H,H], qkv_b, o, o_b, fc1, fc1_b, fc2,
    fc2_b, ln1_w, ln1_b, ln2_w, ln2_b); K_prev/V_prev: per-request [L_b, Hkv, d] bits of the
    cached tokens. Returns (x_out, k_new, v_new) in float64."""
    f = {k: bf16_to_f64(v) for k, v in p.items()}
    B, H = x.shape
    d = H // n_heads
    h = layernorm(x, f["ln1_w"], f["ln1_b"], eps)
    qkv = h @ f["qkv"].T + f["qkv_b"]
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]
    a = np.zeros((B, H))
    for b in range(B):
        K = np.concatenate([bf16_to_f64(K_prev[b]).reshape(-1, H), k[b:b + 1]], axis=0)
        V = np.concatenate([bf16_to_f64(V_prev[b]).reshape(-1, H), v[b:b + 1]], axis=0)
        for hh in range(n_heads):
            sl = slice(hh * d, (hh + 1) * d)
            s = K[:, sl] @ q[b, sl] / math.sqrt(d)
            w = np.exp(s - s.max())
            a[b, sl] = (w / w.sum()) @ V[:, sl]
    x = x + a @ f["o"].T + f["o_b"]
    h = layernorm(x, f["ln2_w"], f["ln2_b"], eps)
    x = x + np.maximum(h @ f["fc1"].T + f["fc1_b"], 0.0) @ f["fc2"].T + f["fc2_b"]
    return x, k.reshape(B, n_heads, d), v.reshape(B, n_heads, d)


def opt_decode_step(tokens, positions, params: dict, K_cache: list, V_cache: list, n_heads: int, eps: float = 1e-5):
    """Full decode step: embeddings (learned positions, offset 2) -> layers -> LN_f -> tied head.
    K_cache[l][b] / V_cache[l][b]: [L_b, Hkv, d] bits of layer l. Returns (logits, x) float64."""
    E = bf16_to_f64(params["embed"])
    P = bf16_to_f64(params["pos"])
    x = E[np.asarray(tokens)] + P[np.asarray(positions) + 2]
    for l in range(len(K_cache)):
        lp = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"L{l}.")}
        x, _, _ = opt_decode_layer(x, lp, K_cache[l], V_cache[l], n_heads, eps)
    h = layernorm(x, bf16_to_f64(params["lnf_w"]), bf16_to_f64(params["lnf_b"]), eps)
    return h @ E.T, x
