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

from .kernels import bf16_to_f64, layernorm, rmsnorm


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


# ------------------------------------------------------------------------------------------------
# Llama family (BASELINE.json configs[2]: Llama-3-70B, TP8 over 8 B200). Pre-RMSNorm, no biases,
# rotary positions (rotate-half convention, theta 500000 for Llama 3), GQA attention, SwiGLU MLP,
# untied LM head. The split operators replace nn.Linear / SDPA as in the paper.

def rope(x, pos: int, theta: float):
    """Rotary embedding of x [..., d] at position pos: (x1, x2) -> (x1 c - x2 s, x2 c + x1 s) with
    angle pos / theta^(2i/d), i < d/2 (Llama's rotate_half layout)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    half = d // 2
    ang = pos * theta ** (-2.0 * np.arange(half) / d)
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


def llama_decode_layer(x, p: dict, K_prev: list, V_prev: list, positions, n_heads: int, n_kv: int,
                       theta: float = 500000.0, eps: float = 1e-5, shard=None):
    """One Llama layer for the new token of every request. x: float64 [B, H]; p: bf16-bit params
    (q [Hq d, H], k, v [Hkv d, H], o [H, Hq d], gate, up [F, H], down [H, F], ln1_w, ln2_w);
    K_prev/V_prev: per-request [L_b, Hkv, d] bits of the cached (already rotated) keys / values.
    shard=(rank, world): compute only tensor-parallel rank `rank`'s heads / FFN rows (Megatron
    column split of q/k/v/gate/up, row split of o/down) and return its PARTIAL o / down outputs
    (without the residual), which the caller sums over ranks (the all-reduce). Returns
    (x_out or (attn_partial, mlp_fn), k_new_roped, v_new)."""
    f = {k: bf16_to_f64(v) for k, v in p.items()}
    B, H = x.shape
    d = f["q"].shape[0] // n_heads
    G = n_heads // n_kv
    h = rmsnorm(x, f["ln1_w"], eps)
    q = (h @ f["q"].T).reshape(B, n_heads, d)
    k = (h @ f["k"].T).reshape(B, n_kv, d)
    v = (h @ f["v"].T).reshape(B, n_kv, d)
    for b in range(B):
        q[b] = rope(q[b], int(positions[b]), theta)
        k[b] = rope(k[b], int(positions[b]), theta)
    heads = range(n_heads) if shard is None else range(shard[0] * n_heads // shard[1], (shard[0] + 1) * n_heads // shard[1])
    a = np.zeros((B, n_heads * d))
    for b in range(B):
        K = np.concatenate([bf16_to_f64(K_prev[b]), k[b:b + 1]], axis=0)  # [L+1, Hkv, d]
        V = np.concatenate([bf16_to_f64(V_prev[b]), v[b:b + 1]], axis=0)
        for hh in heads:
            g = hh // G
            s = K[:, g] @ q[b, hh] / math.sqrt(d)
            w = np.exp(s - s.max())
            a[b, hh * d:(hh + 1) * d] = (w / w.sum()) @ V[:, g]

    def mlp(xx, part=None):
        hm = rmsnorm(xx, f["ln2_w"], eps)
        F = f["gate"].shape[0]
        rows = slice(None) if part is None else slice(part[0] * F // part[1], (part[0] + 1) * F // part[1])
        act = silu(hm @ f["gate"][rows].T) * (hm @ f["up"][rows].T)
        return act @ f["down"][:, rows].T

    if shard is not None:
        cols = slice(heads.start * d, heads.stop * d)
        return (a[:, cols] @ f["o"][:, cols].T, lambda xx: mlp(xx, shard)), k, v
    x = x + a @ f["o"].T
    x = x + mlp(x)
    return x, k, v


def llama_decode_layer_tp(x, p: dict, K_prev: list, V_prev: list, positions, n_heads: int, n_kv: int, world: int,
                          theta: float = 500000.0, eps: float = 1e-5):
    """The same layer computed as `world` tensor-parallel shards whose o / down partials are summed
    in rank order (the all-reduce) before each residual add."""
    parts = [llama_decode_layer(x, p, K_prev, V_prev, positions, n_heads, n_kv, theta, eps, shard=(r, world))
             for r in range(world)]
    x = x + sum(pt[0][0] for pt in parts)
    x = x + sum(pt[0][1](x) for pt in parts)
    return x, parts[0][1], parts[0][2]


def llama_decode_step(tokens, positions, params: dict, K_cache: list, V_cache: list, n_heads: int, n_kv: int,
                      theta: float = 500000.0, eps: float = 1e-5):
    """Embedding -> layers -> final RMSNorm -> LM head (untied). Returns (logits, x) float64."""
    x = bf16_to_f64(params["embed"])[np.asarray(tokens)]
    for l in range(len(K_cache)):
        lp = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"L{l}.")}
        x, _, _ = llama_decode_layer(x, lp, K_cache[l], V_cache[l], positions, n_heads, n_kv, theta, eps)
    h = rmsnorm(x, bf16_to_f64(params["lnf_w"]), eps)
    return h @ bf16_to_f64(params["lm_head"]).T, x


def opt_decode_steps(tokens_seq, start_pos: int, params: dict, K_cache: list, V_cache: list, n_heads: int,
                     eps: float = 1e-5):
    """Several decode steps with teacher forcing: step s feeds tokens_seq[s] at position
    start_pos + s and appends each layer's new k / v to the cache (stored as bf16, the KV cache's
    storage type). Returns the list of per-step logits (float64)."""
    from .kernels import bf16_bits_rne
    L = len(K_cache)
    K = [[np.asarray(k) for k in layer] for layer in K_cache]
    V = [[np.asarray(v) for v in layer] for layer in V_cache]
    E = bf16_to_f64(params["embed"])
    P = bf16_to_f64(params["pos"])
    out = []
    for s, toks in enumerate(tokens_seq):
        toks = np.asarray(toks)
        B = toks.shape[0]
        x = E[toks] + P[np.full(B, start_pos + s) + 2]
        for l in range(L):
            lp = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"L{l}.")}
            x, k_new, v_new = opt_decode_layer(x, lp, K[l], V[l], n_heads, eps)
            for b in range(B):
                kb = bf16_bits_rne(k_new[b])[None]
                vb = bf16_bits_rne(v_new[b])[None]
                K[l][b] = np.concatenate([K[l][b], kb], axis=0)
                V[l][b] = np.concatenate([V[l][b], vb], axis=0)
        h = layernorm(x, bf16_to_f64(params["lnf_w"]), bf16_to_f64(params["lnf_b"]), eps)
        out.append(h @ E.T)
    return out
