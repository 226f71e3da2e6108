"""Tensor-parallel sharding of a Llama decoder (Megatron layout; BASELINE north_star: TP over
8 x B200). Host-side setup logic only (which rows / columns of each weight a rank owns):

- column-parallel (split output rows, no exchange): q, k, v by heads; gate, up by FFN rows;
  the LM head by vocabulary rows (each rank produces its logits shard);
- row-parallel (split input columns): o by q-head columns, down by FFN columns -> every rank
  holds a partial [B, H] output that dak_allreduce_residual sums over ranks (NCCL);
- replicated: RMSNorm weights, token embedding.

Works on any array type supporting 2-D slicing (numpy bf16 bit arrays or torch tensors).
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> slice:
    if n % world:
        raise ValueError(f"{n} is not divisible by the tensor-parallel world {world}")
    k = n // world
    return slice(rank * k, (rank + 1) * k)


def shard_llama(params: dict, rank: int, world: int, n_heads: int, n_kv: int, head_dim: int) -> dict:
    """Full logical parameters (names L{l}.q/k/v/o/gate/up/down/ln1_w/ln2_w, embed, lnf_w, lm_head)
    -> this rank's shard under the same names."""
    out = {}
    for name, w in params.items():
        key = name.split(".", 1)[1] if name.startswith("L") and "." in name else name
        if key == "q":
            out[name] = w[shard_range(n_heads, rank, world).start * head_dim:shard_range(n_heads, rank, world).stop * head_dim]
        elif key in ("k", "v"):
            r = shard_range(n_kv, rank, world)
            out[name] = w[r.start * head_dim:r.stop * head_dim]
        elif key == "o":
            r = shard_range(n_heads, rank, world)
            out[name] = w[:, r.start * head_dim:r.stop * head_dim]
        elif key in ("gate", "up"):
            out[name] = w[shard_range(w.shape[0], rank, world)]
        elif key == "down":
            out[name] = w[:, shard_range(w.shape[1], rank, world)]
        elif key == "lm_head":
            out[name] = w[shard_range(w.shape[0], rank, world)]
        else:  # ln*_w, embed, lnf_w
            out[name] = w
    return out


def local_dims(n_heads: int, n_kv: int, ffn: int, vocab: int, world: int) -> dict:
    for n in (n_heads, n_kv, ffn, vocab):
        if n % world:
            raise ValueError(f"{n} is not divisible by the tensor-parallel world {world}")
    return dict(n_heads=n_heads // world, n_kv=n_kv // world, ffn=ffn // world, vocab=vocab // world)
