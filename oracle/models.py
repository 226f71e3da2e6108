"""Model operator lists and footprints for the planner (TEST INFRASTRUCTURE).

Follows the paper's accounting: decode reads all weights and the KV cache each token;
offloadable ops are the linear layers (weights) and attention (KV) (P:L981 footnote);
C is the weight bytes (linear) or KV bytes (attention) (P:L422 footnote); linear FLOPs are
2*tokens*in*out and decode attention FLOPs are 2*2*B*L*H*d.
Model shapes: OPT-30B and Llama-3-70B (BASELINE.json configs[2]).

Pins (tests/test_oracle_models.py): the shapes and parameter bytes against the Hugging Face
transformers OPT / Llama modules built on the meta device, the FLOP formulas against
torch.utils.flop_counter on the same operations, the KV bytes per token against the cache
tensors a transformers model actually allocates, and the SURVEY a1/a2 totals.

decode_ops is the oracle twin of the C ABI's dak_decode_ops (include/dak.h): same op order, same
integer unit definitions (readings R8, R15, R18 of DESIGN.md) and the same IEEE double operation
order for the FLOPs and T values.
"""
from __future__ import annotations

OPT_30B = dict(name="opt-30b", family="opt", n_layers=48, hidden=7168, n_heads=56, n_kv_heads=56, head_dim=128,
               ffn=28672, vocab=50272, max_pos=2048, dtype_bytes=2, norm="layernorm", act="relu")
LLAMA3_70B = dict(name="llama-3-70b", family="llama", n_layers=80, hidden=8192, n_heads=64, n_kv_heads=8,
                  head_dim=128, ffn=28672, vocab=128256, max_pos=131072, dtype_bytes=2, norm="rmsnorm", act="silu")


def linear_shapes(model: dict, tp: int = 1, fused_qkv: bool = False, fused_gate_up: bool = False):
    """(name, M_out, K_in) of the per-layer linear ops of one TP shard (Megatron split:
    q/k/v/gate/up column-parallel, o/down row-parallel), in model order."""
    h, d = model["hidden"], model["head_dim"]
    for n in (model["n_heads"], model["n_kv_heads"], model["ffn"], model["vocab"]):
        if n % tp:
            raise ValueError("dims must divide by tp")
    hq = model["n_heads"] // tp * d
    hkv = model["n_kv_heads"] // tp * d
    f = model["ffn"] // tp
    qkv = [("qkv", hq + 2 * hkv, h)] if fused_qkv else [("q", hq, h), ("k", hkv, h), ("v", hkv, h)]
    if model["act"] == "relu":  # OPT: q,k,v,o, fc1, fc2
        return qkv + [("o", h, hq), ("fc1", f, h), ("fc2", h, f)]
    gu = [("gate_up", 2 * f, h)] if fused_gate_up else [("gate", f, h), ("up", f, h)]
    return qkv + [("o", h, hq)] + gu + [("down", h, f)]


def linear_weight_bytes(model: dict, tp: int = 1) -> int:
    """Bytes of every decoder layer's linear weights (one shard)."""
    return model["dtype_bytes"] * model["n_layers"] * sum(M * K for _, M, K in linear_shapes(model, tp))


def weight_bytes(model: dict) -> int:
    """Linear + embedding weight bytes (biases and norms are < 0.01% and excluded)."""
    return linear_weight_bytes(model) + model["dtype_bytes"] * model["vocab"] * model["hidden"]


def kv_bytes_per_token(model: dict, tp: int = 1) -> int:
    """K and V rows of one token over all layers: 2 x layers x kv heads x d x dtype."""
    return 2 * model["n_layers"] * (model["n_kv_heads"] // tp) * model["head_dim"] * model["dtype_bytes"]


ROLE = dict(q=0, k=1, v=2, qkv=3, o=4, up=5, fc1=5, down=6, fc2=6, gate=7, gate_up=8, attn=9, head=10)


def decode_ops(model: dict, batch: int, context: int, peak_linear: float, peak_attn: float,
               tp: int = 1, unit_rows: int = 16, chunk_tokens: int = 1024, include_head: bool = True,
               fused_qkv: bool = False, fused_gate_up: bool = False):
    """Per-op planner inputs for one decode step, the definition dak_decode_ops follows.

    Order: per layer its linear ops (model order) then its attention op; the LM head last.
    Linear: C = 2MK; units of unit_rows rows: n = ceil(M/unit_rows), unit_bytes = 2 unit_rows K;
    flops = 2 B M K; T = flops / peak_linear.
    Attention (new token of `batch` requests over `context` cached tokens, this shard's kv heads):
    C = 2 (K and V) * Hkv d * 2 B * batch * context; units = split-KV chunks of chunk_tokens tokens
    of one request: n = batch * ceil(context/chunk_tokens), unit_bytes = ceil(C/n) (reading R15);
    flops = 4 B context (Hq d); T = flops / peak_attn.
    Returns dicts: name, layer, role, kind, M, K, total_bytes, n_units, unit_bytes, flops, T.
    """
    ops = []
    db = model["dtype_bytes"]
    hq = model["n_heads"] // tp * model["head_dim"]
    hkv = model["n_kv_heads"] // tp * model["head_dim"]
    shapes = linear_shapes(model, tp, fused_qkv, fused_gate_up)

    def lin(layer, name, M, K):
        flops = 2.0 * float(batch) * float(M) * float(K)
        ops.append(dict(name=(f"L{layer}.{name}" if layer >= 0 else name), layer=layer, role=ROLE[name],
                        kind="linear", M=M, K=K, total_bytes=M * K * db, n_units=-(-M // unit_rows),
                        unit_bytes=unit_rows * K * db, flops=flops, T=flops / peak_linear))

    for layer in range(model["n_layers"]):
        for name, M, K in shapes:
            lin(layer, name, M, K)
        C = 2 * hkv * db * batch * context
        n = batch * (-(-context // chunk_tokens))
        flops = 4.0 * float(batch) * float(context) * float(hq)
        ops.append(dict(name=f"L{layer}.attn", layer=layer, role=ROLE["attn"], kind="attention",
                        M=batch * context, K=model["head_dim"], total_bytes=C, n_units=n,
                        unit_bytes=-(-C // n), flops=flops, T=flops / peak_attn))
    if include_head:
        lin(-1, "head", model["vocab"] // tp, model["hidden"])
    return ops
