"""Pin the OPT decode-step oracle (oracle/layer.py) against an independent implementation: the
Hugging Face transformers OPT model in float64, fed the same parameters and the same KV cache."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly


def make_params(g, L, H, F, V, maxpos):
    p = {}
    for l in range(L):
        p[f"L{l}.qkv"] = synth.normal_bf16(g, (3 * H, H), 1 / np.sqrt(H))
        p[f"L{l}.qkv_b"] = synth.normal_bf16(g, (3 * H,), 0.1)
        p[f"L{l}.o"] = synth.normal_bf16(g, (H, H), 1 / np.sqrt(H))
        p[f"L{l}.o_b"] = synth.normal_bf16(g, (H,), 0.1)
        p[f"L{l}.fc1"] = synth.normal_bf16(g, (F, H), 1 / np.sqrt(H))
        p[f"L{l}.fc1_b"] = synth.normal_bf16(g, (F,), 0.1)
        p[f"L{l}.fc2"] = synth.normal_bf16(g, (H, F), 1 / np.sqrt(F))
        p[f"L{l}.fc2_b"] = synth.normal_bf16(g, (H,), 0.1)
        for n in ("ln1", "ln2"):
            p[f"L{l}.{n}_w"] = synth.bf16_bits(1.0 + 0.1 * g.standard_normal(H).astype(np.float32))
            p[f"L{l}.{n}_b"] = synth.normal_bf16(g, (H,), 0.1)
    p["embed"] = synth.normal_bf16(g, (V, H), 1.0)
    p["pos"] = synth.normal_bf16(g, (maxpos + 2, H), 0.5)
    p["lnf_w"] = synth.bf16_bits(1.0 + 0.1 * g.standard_normal(H).astype(np.float32))
    p["lnf_b"] = synth.normal_bf16(g, (H,), 0.1)
    return p


def test_opt_decode_step_matches_transformers_float64():
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    from transformers import OPTConfig, OPTForCausalLM
    from transformers.cache_utils import DynamicCache
    L, H, F, V, heads, B, Lp, maxpos = 2, 256, 512, 100, 2, 2, 5, 64
    g = np.random.default_rng(123)
    p = make_params(g, L, H, F, V, maxpos)
    Kc = [[synth.normal_bf16(g, (Lp, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (Lp, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    tokens = np.array([7, 42])
    positions = np.array([Lp, Lp])
    logits, _ = Ly.opt_decode_step(tokens, positions, p, Kc, Vc, heads)

    cfg = OPTConfig(vocab_size=V, hidden_size=H, num_hidden_layers=L, ffn_dim=F, num_attention_heads=heads,
                    max_position_embeddings=maxpos, word_embed_proj_dim=H, do_layer_norm_before=True,
                    enable_bias=True, activation_function="relu", dropout=0.0, attention_dropout=0.0)
    m = OPTForCausalLM(cfg).double().eval()
    f = lambda k: torch.from_numpy(Kx.bf16_to_f64(p[k]))
    sd = {"model.decoder.embed_tokens.weight": f("embed"), "model.decoder.embed_positions.weight": f("pos"),
          "model.decoder.final_layer_norm.weight": f("lnf_w"), "model.decoder.final_layer_norm.bias": f("lnf_b"),
          "lm_head.weight": f("embed")}
    for l in range(L):
        pre = f"model.decoder.layers.{l}."
        W, b = f(f"L{l}.qkv"), f(f"L{l}.qkv_b")
        for i, n in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[pre + f"self_attn.{n}.weight"] = W[i * H:(i + 1) * H]
            sd[pre + f"self_attn.{n}.bias"] = b[i * H:(i + 1) * H]
        sd[pre + "self_attn.out_proj.weight"], sd[pre + "self_attn.out_proj.bias"] = f(f"L{l}.o"), f(f"L{l}.o_b")
        sd[pre + "fc1.weight"], sd[pre + "fc1.bias"] = f(f"L{l}.fc1"), f(f"L{l}.fc1_b")
        sd[pre + "fc2.weight"], sd[pre + "fc2.bias"] = f(f"L{l}.fc2"), f(f"L{l}.fc2_b")
        sd[pre + "self_attn_layer_norm.weight"], sd[pre + "self_attn_layer_norm.bias"] = f(f"L{l}.ln1_w"), f(f"L{l}.ln1_b")
        sd[pre + "final_layer_norm.weight"], sd[pre + "final_layer_norm.bias"] = f(f"L{l}.ln2_w"), f(f"L{l}.ln2_b")
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    cache = DynamicCache()
    for l in range(L):
        k = torch.from_numpy(np.stack([Kx.bf16_to_f64(Kc[l][b]) for b in range(B)])).permute(0, 2, 1, 3)
        v = torch.from_numpy(np.stack([Kx.bf16_to_f64(Vc[l][b]) for b in range(B)])).permute(0, 2, 1, 3)
        cache.update(k.contiguous(), v.contiguous(), l)
    with torch.no_grad():
        out = m(input_ids=torch.from_numpy(tokens).view(B, 1), past_key_values=cache,
                attention_mask=torch.ones(B, Lp + 1, dtype=torch.long),
                position_ids=torch.from_numpy(positions).view(B, 1), use_cache=True)
    ref = out.logits[:, -1].numpy()
    assert np.allclose(logits, ref, rtol=1e-9, atol=1e-9), np.abs(logits - ref).max()


def _hf_opt(p, L, H, F, V, heads, maxpos):
    import torch
    from transformers import OPTConfig, OPTForCausalLM
    cfg = OPTConfig(vocab_size=V, hidden_size=H, num_hidden_layers=L, ffn_dim=F, num_attention_heads=heads,
                    max_position_embeddings=maxpos, word_embed_proj_dim=H, do_layer_norm_before=True,
                    enable_bias=True, activation_function="relu", dropout=0.0, attention_dropout=0.0)
    m = OPTForCausalLM(cfg).double().eval()
    f = lambda k: torch.from_numpy(Kx.bf16_to_f64(p[k]))
    sd = {"model.decoder.embed_tokens.weight": f("embed"), "model.decoder.embed_positions.weight": f("pos"),
          "model.decoder.final_layer_norm.weight": f("lnf_w"), "model.decoder.final_layer_norm.bias": f("lnf_b"),
          "lm_head.weight": f("embed")}
    for l in range(L):
        pre = f"model.decoder.layers.{l}."
        W, b = f(f"L{l}.qkv"), f(f"L{l}.qkv_b")
        for i, n in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[pre + f"self_attn.{n}.weight"] = W[i * H:(i + 1) * H]
            sd[pre + f"self_attn.{n}.bias"] = b[i * H:(i + 1) * H]
        sd[pre + "self_attn.out_proj.weight"], sd[pre + "self_attn.out_proj.bias"] = f(f"L{l}.o"), f(f"L{l}.o_b")
        sd[pre + "fc1.weight"], sd[pre + "fc1.bias"] = f(f"L{l}.fc1"), f(f"L{l}.fc1_b")
        sd[pre + "fc2.weight"], sd[pre + "fc2.bias"] = f(f"L{l}.fc2"), f(f"L{l}.fc2_b")
        sd[pre + "self_attn_layer_norm.weight"], sd[pre + "self_attn_layer_norm.bias"] = f(f"L{l}.ln1_w"), f(f"L{l}.ln1_b")
        sd[pre + "final_layer_norm.weight"], sd[pre + "final_layer_norm.bias"] = f(f"L{l}.ln2_w"), f(f"L{l}.ln2_b")
    _, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    return m


def test_opt_decode_steps_matches_transformers_with_bf16_cache():
    """oracle.layer.opt_decode_steps (teacher-forced multi-step decode, KV stored as bf16) against
    transformers OPT in float64 stepping with a DynamicCache, where after every step the newly
    appended K / V rows are rounded to bf16 by torch (the cache's storage type), independently of
    the oracle's own bf16 rounding."""
    torch = pytest.importorskip("torch")
    pytest.importorskip("transformers")
    from transformers.cache_utils import DynamicCache
    L, H, F, V, heads, B, Lp, maxpos, steps = 2, 128, 256, 97, 2, 2, 6, 64, 4
    g = np.random.default_rng(321)
    p = make_params(g, L, H, F, V, maxpos)
    Kc = [[synth.normal_bf16(g, (Lp, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (Lp, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    toks = [np.array([3 + 5 * s, 40 + 7 * s]) for s in range(steps)]
    ref = Ly.opt_decode_steps(toks, Lp, p, Kc, Vc, heads)
    m = _hf_opt(p, L, H, F, V, heads, maxpos)
    cache = DynamicCache()
    for l in range(L):
        k = torch.from_numpy(np.stack([Kx.bf16_to_f64(Kc[l][b]) for b in range(B)])).permute(0, 2, 1, 3)
        v = torch.from_numpy(np.stack([Kx.bf16_to_f64(Vc[l][b]) for b in range(B)])).permute(0, 2, 1, 3)
        cache.update(k.contiguous(), v.contiguous(), l)
    for s in range(steps):
        with torch.no_grad():
            out = m(input_ids=torch.from_numpy(toks[s]).view(B, 1), past_key_values=cache,
                    attention_mask=torch.ones(B, Lp + s + 1, dtype=torch.long),
                    position_ids=torch.full((B, 1), Lp + s), use_cache=True)
        cache = out.past_key_values
        for layer in cache.layers:  # the step's new rows -> bf16 (RNE, torch's own conversion)
            layer.keys[:, :, -1] = layer.keys[:, :, -1].to(torch.bfloat16).double()
            layer.values[:, :, -1] = layer.values[:, :, -1].to(torch.bfloat16).double()
        got = out.logits[:, -1].numpy()
        assert np.allclose(ref[s], got, rtol=1e-9, atol=1e-9), (s, np.abs(ref[s] - got).max())
    # step 0 of the multi-step oracle is the single-step oracle (pinned above)
    ref_f64 = Ly.opt_decode_step(toks[0], np.full(B, Lp), p, Kc, Vc, heads)[0]
    assert np.allclose(ref_f64, ref[0], rtol=1e-12, atol=1e-12)
