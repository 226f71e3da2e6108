"""Pin oracle/models.py (op shapes, weight / KV bytes, FLOP formulas, decode op list) against
things other than itself: the Hugging Face transformers OPT / Llama modules (parameter shapes on the
meta device, the KV cache tensors a real forward allocates), torch.utils.flop_counter on the
operations the definitions describe, and the SURVEY §8(a) a1/a2 totals (PAPER P:L383-388,
P:L422 footnote)."""
import numpy as np
import pytest

from oracle import models

torch = pytest.importorskip("torch")
tf = pytest.importorskip("transformers")


def _meta_model(mod, layers=2):
    from transformers import LlamaConfig, LlamaForCausalLM, OPTConfig, OPTForCausalLM
    with torch.device("meta"):
        if mod["family"] == "opt":
            return OPTForCausalLM(OPTConfig(hidden_size=mod["hidden"], ffn_dim=mod["ffn"], num_hidden_layers=layers,
                                            num_attention_heads=mod["n_heads"], vocab_size=mod["vocab"],
                                            max_position_embeddings=mod["max_pos"], word_embed_proj_dim=mod["hidden"]))
        return LlamaForCausalLM(LlamaConfig(hidden_size=mod["hidden"], intermediate_size=mod["ffn"],
                                            num_hidden_layers=layers, num_attention_heads=mod["n_heads"],
                                            num_key_value_heads=mod["n_kv_heads"], vocab_size=mod["vocab"],
                                            head_dim=mod["head_dim"], tie_word_embeddings=False))


HF_NAMES = dict(q="self_attn.q_proj", k="self_attn.k_proj", v="self_attn.v_proj", fc1="fc1", fc2="fc2",
                gate="mlp.gate_proj", up="mlp.up_proj", down="mlp.down_proj")


@pytest.mark.parametrize("name", ["OPT_30B", "LLAMA3_70B"])
def test_linear_shapes_match_transformers(name):
    """Every per-layer linear of the oracle has the [out, in] shape of the transformers module, and
    the set of decoder Linear modules is exactly the oracle's list (the paper's offloadable linear
    ops, P:L981 footnote)."""
    mod = getattr(models, name)
    m = _meta_model(mod)
    layer = (m.model.decoder.layers[0] if mod["family"] == "opt" else m.model.layers[0])
    lin = {n: tuple(p.weight.shape) for n, p in layer.named_modules() if isinstance(p, torch.nn.Linear)}
    names = dict(HF_NAMES, o="self_attn.out_proj" if mod["family"] == "opt" else "self_attn.o_proj")
    shapes = models.linear_shapes(mod)
    assert sorted(names[n] for n, _, _ in shapes) == sorted(lin)
    for n, M, K in shapes:
        assert lin[names[n]] == (M, K), n
    # fused forms (reading R18) stack the same rows
    fq = models.linear_shapes(mod, fused_qkv=True, fused_gate_up=True)
    assert fq[0] == ("qkv", sum(M for n, M, _ in shapes if n in "qkv"), mod["hidden"])


@pytest.mark.parametrize("name", ["OPT_30B", "LLAMA3_70B"])
def test_weight_bytes_match_transformers_params(name):
    """linear_weight_bytes = 2 B x the parameter count of every decoder Linear weight of the
    transformers model (2 layers, scaled to n_layers); weight_bytes adds the token embedding."""
    mod = getattr(models, name)
    m = _meta_model(mod, layers=2)
    layers = m.model.decoder.layers if mod["family"] == "opt" else m.model.layers
    per_layer = sum(p.weight.numel() for p in layers[0].modules() if isinstance(p, torch.nn.Linear))
    assert models.linear_weight_bytes(mod) == 2 * per_layer * mod["n_layers"]
    emb = (m.model.decoder.embed_tokens if mod["family"] == "opt" else m.model.embed_tokens).weight.numel()
    assert models.weight_bytes(mod) == 2 * (per_layer * mod["n_layers"] + emb)


def test_survey_a1_a2_totals():
    """SURVEY §8(a) a1/a2 numbers: OPT-30B linear weights 59.19e9 B, q/k/v/o 102,760,448 B and
    fc1/fc2 411,041,792 B per op; Llama-3-70B 141.1e9 B of weights (with both embeddings) and a
    TP8 shard of 213.9 MB per GPU per layer; KV 1,376,256 / 327,680 B per token (40,960 B per
    token per GPU at TP8)."""
    opt, ll = models.OPT_30B, models.LLAMA3_70B
    assert round(models.linear_weight_bytes(opt) / 1e9, 2) == 59.19
    sh = dict((n, M * K * 2) for n, M, K in models.linear_shapes(opt))
    assert sh["q"] == sh["k"] == sh["v"] == sh["o"] == 102_760_448
    assert sh["fc1"] == sh["fc2"] == 411_041_792
    full = models.linear_weight_bytes(ll) + 2 * 2 * ll["vocab"] * ll["hidden"]  # untied embed + head
    assert round(full / 1e9, 1) == 141.1
    per_gpu_layer = models.linear_weight_bytes(ll, tp=8) / ll["n_layers"]
    assert round(per_gpu_layer / 1e6, 1) == 213.9
    assert models.linear_weight_bytes(ll, tp=8) * 8 == models.linear_weight_bytes(ll)  # sharding keeps bytes
    assert models.kv_bytes_per_token(opt) == 1_376_256
    assert models.kv_bytes_per_token(ll) == 327_680 and models.kv_bytes_per_token(ll, tp=8) == 40_960


@pytest.mark.parametrize("family", ["opt", "llama"])
def test_kv_bytes_match_transformers_cache(family):
    """KV bytes per token = what a transformers model's cache actually holds after a bf16 forward
    (tiny model of the same structure; GQA for Llama), and the attention op's C_i is that times
    batch x context."""
    from transformers import LlamaConfig, LlamaForCausalLM, OPTConfig, OPTForCausalLM
    torch.manual_seed(0)
    if family == "opt":
        mod = dict(models.OPT_30B, n_layers=3, hidden=64, n_heads=4, n_kv_heads=4, head_dim=16, ffn=128, vocab=50)
        m = OPTForCausalLM(OPTConfig(hidden_size=64, ffn_dim=128, num_hidden_layers=3, num_attention_heads=4,
                                     vocab_size=50, max_position_embeddings=64, word_embed_proj_dim=64))
    else:
        mod = dict(models.LLAMA3_70B, n_layers=3, hidden=64, n_heads=8, n_kv_heads=2, head_dim=8, ffn=128, vocab=50)
        m = LlamaForCausalLM(LlamaConfig(hidden_size=64, intermediate_size=128, num_hidden_layers=3,
                                         num_attention_heads=8, num_key_value_heads=2, vocab_size=50, head_dim=8))
    m = m.to(torch.bfloat16).eval()
    B, L = 3, 11
    with torch.no_grad():
        out = m(input_ids=torch.randint(0, 50, (B, L)), use_cache=True)
    cache = out.past_key_values
    nbytes = 0
    for layer in cache.layers:
        nbytes += layer.keys.numel() * layer.keys.element_size() + layer.values.numel() * layer.values.element_size()
    assert nbytes == models.kv_bytes_per_token(mod) * B * L
    ops = models.decode_ops(mod, B, L, 1e15, 1e15, chunk_tokens=4)
    att = [o for o in ops if o["kind"] == "attention"]
    assert sum(o["total_bytes"] for o in att) == nbytes
    assert att[0]["n_units"] == B * 3 and (att[0]["n_units"] - 1) * att[0]["unit_bytes"] < att[0]["total_bytes"] \
        <= att[0]["n_units"] * att[0]["unit_bytes"]


def test_flops_match_flop_counter():
    """FLOPs of decode_ops = torch.utils.flop_counter's count of the operations the definitions
    describe: F.linear(x [B, K], W [M, K]) and decode attention as q.K^T then p.V per q head
    (GQA: each q head reads its group's kv head)."""
    from torch.utils.flop_counter import FlopCounterMode
    mod = dict(models.LLAMA3_70B, n_layers=1, hidden=64, n_heads=8, n_kv_heads=2, head_dim=16, ffn=96, vocab=40)
    B, L = 3, 10
    ops = models.decode_ops(mod, B, L, 1e15, 1e15)
    for o in ops:
        if o["kind"] == "linear":
            x, W = torch.zeros(B, o["K"]), torch.zeros(o["M"], o["K"])
            with FlopCounterMode(display=False) as fc:
                torch.nn.functional.linear(x, W)
            assert fc.get_total_flops() == o["flops"], o["name"]
        else:
            q = torch.zeros(B, mod["n_heads"], 1, mod["head_dim"])
            K = torch.zeros(B, mod["n_heads"], L, mod["head_dim"])  # kv heads repeated per q head
            with FlopCounterMode(display=False) as fc:
                p = q @ K.transpose(-1, -2)
                _ = p @ K
            assert fc.get_total_flops() == o["flops"]
            assert o["T"] == o["flops"] / 1e15


def test_decode_ops_structure():
    """Op order (per layer: linears then attention; head last), unit rules (R8, R15) and T."""
    mod = models.OPT_30B
    ops = models.decode_ops(mod, 8, 64, 1.3554e15, 1.3554e15, unit_rows=16, chunk_tokens=64, fused_qkv=True)
    assert len(ops) == 48 * 5 + 1
    assert [o["role"] for o in ops[:5]] == [models.ROLE[n] for n in ("qkv", "o", "fc1", "fc2", "attn")]
    assert ops[-1]["name"] == "head" and ops[-1]["M"] == mod["vocab"]
    q = ops[0]
    assert q["n_units"] == 3 * 7168 // 16 and q["unit_bytes"] == 16 * 7168 * 2
    a = ops[4]
    assert a["total_bytes"] == 1_376_256 // 48 * 8 * 64 and a["n_units"] == 8
    total = sum(o["total_bytes"] for o in ops)
    assert total == models.linear_weight_bytes(mod) + 2 * mod["vocab"] * mod["hidden"] + 1_376_256 * 8 * 64
