"""Pins of the Llama decode-step oracle (oracle/layer.py, BASELINE configs[2] model family):
rotary embedding properties, tensor-parallel shard sums, and the whole decode step against the
Hugging Face transformers Llama model fed the same parameters and KV cache."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly


def make_llama_params(g, L, H, F, V, nh, nkv, d):
    p = {}
    for l in range(L):
        p[f"L{l}.q"] = synth.normal_bf16(g, (nh * d, H), 1 / np.sqrt(H))
        p[f"L{l}.k"] = synth.normal_bf16(g, (nkv * d, H), 1 / np.sqrt(H))
        p[f"L{l}.v"] = synth.normal_bf16(g, (nkv * d, H), 1 / np.sqrt(H))
        p[f"L{l}.o"] = synth.normal_bf16(g, (H, nh * d), 1 / np.sqrt(nh * d))
        p[f"L{l}.gate"] = synth.normal_bf16(g, (F, H), 1 / np.sqrt(H))
        p[f"L{l}.up"] = synth.normal_bf16(g, (F, H), 1 / np.sqrt(H))
        p[f"L{l}.down"] = synth.normal_bf16(g, (H, F), 1 / np.sqrt(F))
        for n in ("ln1_w", "ln2_w"):
            p[f"L{l}.{n}"] = synth.bf16_bits(1.0 + 0.1 * g.standard_normal(H).astype(np.float32))
    p["embed"] = synth.normal_bf16(g, (V, H), 1.0)
    p["lnf_w"] = synth.bf16_bits(1.0 + 0.1 * g.standard_normal(H).astype(np.float32))
    p["lm_head"] = synth.normal_bf16(g, (V, H), 1 / np.sqrt(H))
    return p


def test_rope_pins():
    g = synth.rng(5)
    x = g.standard_normal((3, 128))
    assert np.array_equal(Ly.rope(x, 0, 500000.0), x)  # position 0 is the identity
    y = Ly.rope(x, 37, 500000.0)
    # each (i, i + d/2) pair is rotated: pair norms preserved
    assert np.allclose(x[:, :64] ** 2 + x[:, 64:] ** 2, y[:, :64] ** 2 + y[:, 64:] ** 2, rtol=1e-12)
    # relative position: <R(m) q, R(n) k> depends on m - n only
    q, k = g.standard_normal(128), g.standard_normal(128)
    a = Ly.rope(q, 100, 10000.0) @ Ly.rope(k, 90, 10000.0)
    b = Ly.rope(q, 17, 10000.0) @ Ly.rope(k, 7, 10000.0)
    assert np.isclose(a, b, rtol=1e-10)
    # the first pair rotates by exactly pos radians (theta^0 = 1)
    e = np.zeros(128)
    e[0] = 1.0
    r = Ly.rope(e, 2, 500000.0)
    assert np.isclose(r[0], np.cos(2.0)) and np.isclose(r[64], np.sin(2.0))


def test_silu_closed_form():
    assert Ly.silu(np.array([0.0]))[0] == 0.0
    assert np.isclose(Ly.silu(np.array([1.0]))[0], 1.0 / (1.0 + np.exp(-1.0)))
    assert np.isclose(Ly.silu(np.array([-30.0]))[0], -30.0 * np.exp(-30.0), rtol=1e-6)


@pytest.mark.parametrize("world", [2, 4])
def test_tp_shards_sum_to_unsharded(world):
    """Megatron TP: column-split q/k/v/gate/up + row-split o/down, partials summed in rank order,
    equals the unsharded layer (up to float64 rounding)."""
    g = synth.rng(8)
    H, F, nh, nkv, d, B = 256, 384, 8, 4, 32, 3
    p = make_llama_params(g, 1, H, F, 50, nh, nkv, d)
    lp = {k.split(".", 1)[1]: v for k, v in p.items() if k.startswith("L0.")}
    x = g.standard_normal((B, H))
    Kp = [synth.normal_bf16(g, (5 + b, nkv, d)) for b in range(B)]
    Vp = [synth.normal_bf16(g, (5 + b, nkv, d)) for b in range(B)]
    pos = np.array([5, 6, 7])
    ref, k, v = Ly.llama_decode_layer(x, lp, Kp, Vp, pos, nh, nkv)
    tp, k2, v2 = Ly.llama_decode_layer_tp(x, lp, Kp, Vp, pos, nh, nkv, world)
    assert np.allclose(tp, ref, rtol=1e-12, atol=1e-12)
    assert np.array_equal(k, k2) and np.array_equal(v, v2)


def test_llama_decode_step_matches_transformers_float64():
    torch = pytest.importorskip("torch")
    pytest.importorskip("transformers")
    from transformers import LlamaConfig, LlamaForCausalLM
    from transformers.cache_utils import DynamicCache
    L, H, F, V, nh, nkv, d, B, Lp = 2, 256, 512, 100, 4, 2, 64, 2, 6
    g = synth.rng(321)
    p = make_llama_params(g, L, H, F, V, nh, nkv, d)
    Kc = [[synth.normal_bf16(g, (Lp, nkv, d)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (Lp, nkv, d)) for _ in range(B)] for _ in range(L)]
    tokens = np.array([7, 42])
    positions = np.array([Lp, Lp])
    logits, _ = Ly.llama_decode_step(tokens, positions, p, Kc, Vc, nh, nkv)

    cfg = LlamaConfig(vocab_size=V, hidden_size=H, intermediate_size=F, num_hidden_layers=L, num_attention_heads=nh,
                      num_key_value_heads=nkv, head_dim=d, rms_norm_eps=1e-5, rope_theta=500000.0,
                      max_position_embeddings=128, tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    m = LlamaForCausalLM(cfg).double().eval()
    f = lambda k: torch.from_numpy(Kx.bf16_to_f64(p[k]))
    sd = {"model.embed_tokens.weight": f("embed"), "model.norm.weight": f("lnf_w"), "lm_head.weight": f("lm_head")}
    for l in range(L):
        pre = f"model.layers.{l}."
        for n, key in (("q_proj", "q"), ("k_proj", "k"), ("v_proj", "v"), ("o_proj", "o")):
            sd[pre + f"self_attn.{n}.weight"] = f(f"L{l}.{key}")
        for n in ("gate", "up", "down"):
            sd[pre + f"mlp.{n}_proj.weight"] = f(f"L{l}.{n}")
        sd[pre + "input_layernorm.weight"] = f(f"L{l}.ln1_w")
        sd[pre + "post_attention_layernorm.weight"] = f(f"L{l}.ln2_w")
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    cache = DynamicCache()
    for l in range(L):
        Kt = torch.from_numpy(np.stack([Kx.bf16_to_f64(Kc[l][b]) for b in range(B)]).transpose(0, 2, 1, 3).copy())
        Vt = torch.from_numpy(np.stack([Kx.bf16_to_f64(Vc[l][b]) for b in range(B)]).transpose(0, 2, 1, 3).copy())
        cache.update(Kt, Vt, l)
    with torch.no_grad():
        out = m(input_ids=torch.from_numpy(tokens[:, None]), past_key_values=cache,
                position_ids=torch.from_numpy(positions[:, None]), use_cache=True)
    ref = out.logits[:, -1].numpy()
    # transformers computes RMSNorm statistics and the rotary tables in float32 even for float64
    # weights: agreement is at that precision
    assert np.allclose(logits, ref, rtol=2e-5, atol=2e-5), np.abs(logits - ref).max()
