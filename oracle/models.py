"""Model operator lists and footprints for the planner (TEST INFRASTRUCTURE).

Follows the paper's accounting: decode reads all weights and the KV cache each token;
offloadable ops are the linear layers (weights) and attention (KV) (P:L981 footnote);
C is the weight bytes (linear) or KV bytes (attention) (P:L422 footnote); linear FLOPs are
2*tokens*in*out and decode attention FLOPs are 2*2*B*L*H*d.
Model shapes: OPT-30B and Llama-3-70B (BASELINE.json configs[2]).
"""
from __future__ import annotations

OPT_30B = dict(name="opt-30b", n_layers=48, hidden=7168, n_heads=56, n_kv_heads=56, head_dim=128,
               ffn=28672, vocab=50272, max_pos=2048, dtype_bytes=2, norm="layernorm", act="relu")
LLAMA3_70B = dict(name="llama-3-70b", n_layers=80, hidden=8192, n_heads=64, n_kv_heads=8, head_dim=128,
                  ffn=28672, vocab=128256, max_pos=131072, dtype_bytes=2, norm="rmsnorm", act="silu")


def linear_shapes(model: dict, tp: int = 1):
    """(name, M_out, K_in) of the per-layer linear ops of one TP shard (Megatron split:
    q/k/v/gate/up column-parallel, o/down row-parallel)."""
    h, d = model["hidden"], model["head_dim"]
    hq = model["n_heads"] * d // tp
    hkv = model["n_kv_heads"] * d // tp
    f = model["ffn"] // tp
    if model["act"] == "relu":  # OPT: q,k,v,o, fc1, fc2
        return [("q", hq, h), ("k", hkv, h), ("v", hkv, h), ("o", h, hq), ("fc1", f, h), ("fc2", h, f)]
    return [("q", hq, h), ("k", hkv, h), ("v", hkv, h), ("o", h, hq), ("gate", f, h), ("up", f, h), ("down", h, f)]


def weight_bytes(model: dict) -> int:
    """Linear + embedding weight bytes (biases and norms are < 0.01% and excluded)."""
    per_layer = sum(M * K for _, M, K in linear_shapes(model))
    emb = model["vocab"] * model["hidden"]
    return model["dtype_bytes"] * (model["n_layers"] * per_layer + emb)


def decode_ops(model: dict, batch: int, context: int, peak_linear: float, peak_attn: float,
               tp: int = 1, unit_rows: int = 16, attn_unit_tokens: int = 1024, include_head: bool = True):
    """Per-op planner inputs for one decode step.

    Returns a list of dicts: name, kind, M, K, total_bytes, n_units, unit_bytes, flops, T.
    Linear units are `unit_rows` output rows (last unit may be short); attention units are
    split-KV chunks of `attn_unit_tokens` tokens of one request (all kv heads of the shard).
    """
    ops = []
    db = model["dtype_bytes"]
    kvh = model["n_kv_heads"] // tp if model["n_kv_heads"] >= tp else 1
    qh = model["n_heads"] // tp
    d = model["head_dim"]
    for layer in range(model["n_layers"]):
        for name, M, K in linear_shapes(model, tp):
            C = M * K * db
            n_units = -(-M // unit_rows)
            flops = 2.0 * batch * M * K
            ops.append(dict(name=f"L{layer}.{name}", kind="linear", M=M, K=K, total_bytes=C,
                            n_units=n_units, unit_bytes=unit_rows * K * db, flops=flops, T=flops / peak_linear))
        C = 2 * kvh * d * db * batch * context
        chunks_per_req = -(-context // attn_unit_tokens)
        unit_bytes = 2 * kvh * d * db * attn_unit_tokens
        flops = 4.0 * batch * context * qh * d
        ops.append(dict(name=f"L{layer}.attn", kind="attention", M=batch * context, K=d, total_bytes=C,
                        n_units=batch * chunks_per_req, unit_bytes=unit_bytes if chunks_per_req > 1 else C // batch,
                        flops=flops, T=flops / peak_attn))
    if include_head:
        M, K = model["vocab"] // tp, model["hidden"]
        C = M * K * db
        ops.append(dict(name="head", kind="linear", M=M, K=K, total_bytes=C, n_units=-(-M // unit_rows),
                        unit_bytes=unit_rows * K * db, flops=2.0 * batch * M * K, T=2.0 * batch * M * K / peak_linear))
    return ops
