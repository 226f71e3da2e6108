"""GPU parity of the composed decode step (dak_layer x L + embed + LN + LM head via the engine)
against the OPT decode-step oracle (itself pinned to transformers OPT in float64).

Tolerance: the GPU keeps activations in bf16 between kernels (h, qkv, attention output, fc1
output, residual stream), i.e. ~6 sequential roundings of 2^-9 relative per layer; the step is
compared within 3e-2 of max(|ref|, rms(ref))."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly
from tests.test_oracle_layer import make_params

pytestmark = pytest.mark.gpu


def _engine_weights(p, L, torch):
    def dev(bits):
        return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)
    w = {}
    for l in range(L):
        for ours, theirs in (("qkv", "qkv"), ("o", "o"), ("up", "fc1"), ("down", "fc2")):
            w[f"L{l}.{ours}"] = dev(p[f"L{l}.{theirs}"])
            w[f"L{l}.{ours}.b"] = dev(p[f"L{l}.{theirs}_b"])
        for n in ("ln1_w", "ln1_b", "ln2_w", "ln2_b"):
            w[f"L{l}.{n}"] = dev(p[f"L{l}.{n}"])
    for n in ("embed", "pos", "lnf_w", "lnf_b"):
        w[n] = dev(p[n])
    return w


@pytest.mark.parametrize("fuse,fused_qkv", [(True, True), (True, False), (False, True)])
@pytest.mark.parametrize("frac,B,ctx", [(0.0, 3, 70), (0.2, 3, 70), (0.5, 2, 200)])
def test_engine_step_matches_oracle(frac, B, ctx, fuse, fused_qkv):
    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, OPTConfig, HW
    L, H, F, V, heads, maxpos = 2, 256, 512, 1000, 2, 256
    g = np.random.default_rng(2024)
    p = make_params(g, L, H, F, V, maxpos)
    cfg = OPTConfig(n_layers=L, hidden=H, n_heads=heads, ffn=F, vocab=V, max_pos=maxpos, name="opt-tiny")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    total = sum(o for o in [3 * H * H, H * H, F * H, H * F]) * 2 * L + V * H * 2
    eng = DakOPT(cfg, B, ctx, hw, mode=dak.PLAN_EXACT, y_req=int(frac * total), page_size=64, chunk_pages=1,
                 weights=_engine_weights(p, L, torch), fuse_norm=fuse, fused_qkv=fused_qkv)
    if frac > 0:
        assert sum(op.h for op in eng.linear_ops()) > 0
    Kc = [[synth.normal_bf16(g, (ctx - 1, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (ctx - 1, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    tokens = np.arange(B) * 37 + 5
    eng.tokens.copy_(torch.from_numpy(tokens.astype(np.int32)))
    s = torch.cuda.Stream()
    eng.capture(s)  # also runs one eager step (warm-up) before capture
    # the eager step appended the new token already; replaying rewrites the same slot
    eng.graph.replay()
    torch.cuda.synchronize()
    ref, _ = Ly.opt_decode_step(tokens, np.full(B, ctx - 1), p, Kc, Vc, heads)
    got = Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16))
    from tests.gpu_util import assert_close
    assert_close(got, ref, rtol=3e-2)
    eng.close()


@pytest.mark.parametrize("frac", [0.0, 0.3])
def test_engine_multistep_decode_matches_oracle(frac):
    """Four decode steps (teacher-forced tokens) through one captured CUDA graph: each step appends
    its KV row at the next position (crossing a page and a split-KV chunk boundary) and the logits
    of every step match the oracle, which carries its own bf16 KV cache forward."""
    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, OPTConfig, HW
    L, H, F, V, heads, maxpos, B, prompt, steps = 2, 256, 512, 1000, 2, 256, 2, 62, 4
    g = np.random.default_rng(77)
    p = make_params(g, L, H, F, V, maxpos)
    cfg = OPTConfig(n_layers=L, hidden=H, n_heads=heads, ffn=F, vocab=V, max_pos=maxpos, name="opt-tiny")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    total = (4 * H * H + 2 * F * H) * 2 * L + V * H * 2
    eng = DakOPT(cfg, B, prompt + 1, hw, mode=dak.PLAN_EXACT, y_req=int(frac * total), page_size=64, chunk_pages=1,
                 weights=_engine_weights(p, L, torch), max_context=prompt + steps + 1)
    Kc = [[synth.normal_bf16(g, (prompt, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (prompt, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    toks = [np.array([3 + 11 * s, 500 + 7 * s]) for s in range(steps)]
    s_ = torch.cuda.Stream()
    eng.tokens.copy_(torch.from_numpy(toks[0].astype(np.int32)))
    eng.capture(s_)  # eager warm step writes position `prompt` with toks[0]; replay rewrites it
    got = []
    for s in range(steps):
        eng.tokens.copy_(torch.from_numpy(toks[s].astype(np.int32)))
        eng.graph.replay()
        torch.cuda.synchronize()
        got.append(Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16)))
        if s + 1 < steps:
            eng.advance()
            torch.cuda.synchronize()
    ref = Ly.opt_decode_steps(toks, prompt, p, Kc, Vc, heads)
    from tests.gpu_util import assert_close
    for s in range(steps):
        assert_close(got[s], ref[s], rtol=3e-2)
    eng.close()


def test_engine_kv_replan_across_steps_matches_oracle():
    """KV placement across decode steps (reading R23): with kv_replan the engine re-places the KV
    each time the requests open a new split-KV chunk -- the attention ops keep the planner's host
    ratio, dak_kv_replace moves the next-oldest chunks to the host, dak_kv_migrate copies those pages
    on the device, the captured graph reads the rewritten tables. Every step's logits match the
    oracle's multi-step decode, and the block tables after each re-placement equal the oracle's
    chain (kv_place_chunk_major, then kv_replace with kv_host_units_keep_ratio) bit for bit."""
    import torch
    from oracle import partition as Pt
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, OPTConfig, HW
    L, H, F, V, heads, maxpos, B, prompt, steps, page = 2, 256, 512, 1000, 2, 256, 3, 40, 12, 16
    g = np.random.default_rng(78)
    p = make_params(g, L, H, F, V, maxpos)
    cfg = OPTConfig(n_layers=L, hidden=H, n_heads=heads, ffn=F, vocab=V, max_pos=maxpos, name="opt-tiny")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    total = (4 * H * H + 2 * F * H) * 2 * L + V * H * 2
    eng = DakOPT(cfg, B, prompt + 1, hw, mode=dak.PLAN_EXACT, y_req=int(0.45 * total), page_size=page, chunk_pages=1,
                 weights=_engine_weights(p, L, torch), max_context=prompt + steps + 1, kv_replan=True)
    assert min(eng.attn_host_chunks) > 0
    Kc = [[synth.normal_bf16(g, (prompt, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (prompt, heads, H // heads)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    ppr = eng.pages_per_req
    ref_tables = [Pt.kv_place_chunk_major([prompt + 1] * B, page, ppr, 1, eng.attn_host_chunks[l])[0] for l in range(L)]
    n0 = [eng.attn_units[l] for l in range(L)]
    toks = [np.array([3 + 11 * s, 500 + 7 * s, 900 - 5 * s]) for s in range(steps)]
    s_ = torch.cuda.Stream()
    eng.tokens.copy_(torch.from_numpy(toks[0].astype(np.int32)))
    eng.capture(s_)
    got, replans = [], 0
    for s in range(steps):
        eng.tokens.copy_(torch.from_numpy(toks[s].astype(np.int32)))
        eng.graph.replay()
        torch.cuda.synchronize()
        got.append(Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16)))
        if s + 1 < steps:
            eng.advance()
            torch.cuda.synchronize()
            Lc = prompt + s + 2
            if (Lc - 1) % page == 0:  # a new chunk opened: the engine re-placed
                replans += 1
                n_new = B * (-(-Lc // page))
                for l in range(L):
                    hu = Pt.kv_host_units_keep_ratio(eng.attn_host_chunks[l], n0[l], n_new)
                    ref_tables[l], _ = Pt.kv_replace(ref_tables[l], [Lc] * B, page, ppr, 1, hu, B * ppr, B * ppr)
                    dev = eng.block_tables[l].cpu().numpy().view(np.uint32)
                    assert np.array_equal(dev, np.array(ref_tables[l], dtype=np.uint32)), (s, l)
    assert replans >= 1
    host_pages = sum(int(((np.array(t, dtype=np.uint32) & 0x80000000) != 0).sum()) for t in ref_tables)
    assert host_pages > sum(eng.attn_host_chunks)  # the KV moved to the host as it grew
    ref = Ly.opt_decode_steps(toks, prompt, p, Kc, Vc, heads)
    from tests.gpu_util import assert_close
    for s in range(steps):
        assert_close(got[s], ref[s], rtol=3e-2)
    eng.close()


@pytest.mark.parametrize("fused_qkv,ctx,max_ctx,frac", [(True, 70, None, 0.3), (False, 63, 67, 0.3), (True, 200, 260, 0.6)])
def test_engine_plan_and_placement_match_oracle(fused_qkv, ctx, max_ctx, frac):
    """The engine's op list (dak_decode_ops), ratios (dak_plan_ratios) and KV placement
    (dak_kv_place) equal the oracle's definitions bit for bit; the placed host bytes of every
    attention op equal the planned ones up to the short last chunk of each request (reading R15),
    and the step's host-byte accounting is what was placed."""
    import torch
    from oracle import models, partition as Pt, planner as P
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, OPTConfig, HW
    L, H, F, V, heads, maxpos, B = 2, 256, 512, 1000, 2, 256, 3
    cfg = OPTConfig(n_layers=L, hidden=H, n_heads=heads, ffn=F, vocab=V, max_pos=maxpos, name="opt-tiny")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    mod = dict(models.OPT_30B, n_layers=L, hidden=H, n_heads=heads, n_kv_heads=heads, head_dim=H // heads, ffn=F,
               vocab=V)
    total = sum(o["total_bytes"] for o in models.decode_ops(mod, B, ctx, 1, 1))
    y = int(frac * total)
    eng = DakOPT(cfg, B, ctx, hw, mode=dak.PLAN_EXACT, y_req=y, page_size=64, chunk_pages=1, fused_qkv=fused_qkv,
                 max_context=max_ctx)
    ref_ops = models.decode_ops(mod, B, ctx, hw.peak_flops, hw.peak_flops, unit_rows=16, chunk_tokens=64,
                                fused_qkv=fused_qkv)
    assert len(eng.plan_ops) == len(ref_ops)
    for g_, r_ in zip(eng.plan_ops, ref_ops):
        for f in ("n_units", "unit_bytes", "total_bytes", "M", "K", "T"):
            assert g_[f] == r_[f]
    ref_plan = P.plan_units(ref_ops, hw.hbm_bps, hw.link_bps, y, dak.PLAN_EXACT)
    assert [p["host_units"] for p in eng.plan] == ref_plan["host_units"]
    att = [i for i, o in enumerate(ref_ops) if o["kind"] == "attention"]
    tok = 2 * heads * (H // heads) * 2
    for l, i in enumerate(att):
        hu = ref_plan["host_units"][i]
        rt, rh, rg, rtok = Pt.kv_place_chunk_major([ctx] * B, 64, eng.pages_per_req, 1, hu)
        assert np.array_equal(eng.block_tables[l].cpu().numpy().view(np.uint32), np.array(rt, dtype=np.uint32))
        assert eng.kv_host_tokens[l] == rtok and eng.kv[l][4] == rh
        planned = ref_plan["host_bytes"][i]
        assert abs(rtok * tok - planned) <= B * 64 * tok  # within one chunk per request (short last chunks)
    nb = eng.bytes_per_step()
    lin_host = sum(op.h * op.K * 2 for op in eng.linear_ops())
    assert nb["host"] == lin_host + tok * sum(eng.kv_host_tokens)
    assert nb["total"] == sum(o["total_bytes"] for o in ref_ops)
    eng.close()
