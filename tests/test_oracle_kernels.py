"""Pins for oracle/kernels.py against textbook identities, exact integer arithmetic and libraries."""
import math

import numpy as np
import pytest

import synth
from oracle import kernels as Kx


def test_bf16_decode_bit_level():
    bits = np.array([0x3F80, 0xBF80, 0x4000, 0x0000, 0x8000, 0x7F80, 0x3F81], dtype=np.uint16)
    v = Kx.bf16_to_f64(bits)
    assert v[0] == 1.0 and v[1] == -1.0 and v[2] == 2.0 and v[3] == 0.0
    assert math.copysign(1, v[4]) == -1 and math.isinf(v[5])
    assert v[6] == 1.0 + 2.0**-7
    # synth rounding (RNE) round trip on representable values
    vals = np.array([1.0, -3.5, 0.15625, 65280.0], dtype=np.float32)
    assert np.array_equal(Kx.bf16_to_f64(synth.bf16_bits(vals)), vals.astype(np.float64))


def test_linear_integer_exact_vs_python_ints():
    """Integer inputs: the float64 result must equal exact integer arithmetic (brute force)."""
    M, K, N = 37, 96, 3
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(0, 1), kind="int", bias=True)
    y = Kx.linear(W, x, bias_bits=b)
    Wi = Kx.bf16_to_f64(W).astype(int)
    xi = Kx.bf16_to_f64(x).astype(int)
    bi = Kx.bf16_to_f64(b).astype(int)
    for n in range(N):
        for m in range(M):
            assert y[n, m] == sum(int(Wi[m, k]) * int(xi[n, k]) for k in range(K)) + int(bi[m])


def test_linear_rowloop_matches_matmul_and_onehot():
    M, K, N = 50, 128, 4
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(0, 2))
    y1 = Kx.linear_rowloop(W, x)
    y2 = Kx.linear(W, x)
    assert np.allclose(y1, y2, rtol=1e-12, atol=1e-12)
    # one-hot x picks out a column of W exactly
    oh = np.zeros((1, K), dtype=np.float32)
    oh[0, 17] = 1.0
    y = Kx.linear(W, synth.bf16_bits(oh))
    assert np.array_equal(y[0], Kx.bf16_to_f64(W)[:, 17])


def test_linear_rank1_closed_form():
    """W = u v^T -> y = u (v . x) (closed form)."""
    g = np.random.default_rng(3)
    u = g.integers(-3, 4, size=40).astype(np.float32)
    v = g.integers(-3, 4, size=64).astype(np.float32)
    x = g.integers(-3, 4, size=(2, 64)).astype(np.float32)
    W = synth.bf16_bits(np.outer(u, v))
    y = Kx.linear(W, synth.bf16_bits(x))
    assert np.array_equal(y, np.outer(x.astype(np.float64) @ v, u))


def test_split_linear_r_invariance_and_epilogue():
    """Result independent of the host/HBM split point h (north star: 'results independent of r')."""
    M, K, N = 64, 256, 2
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(0, 3), bias=True)
    res = synth.normal_bf16(np.random.default_rng(0), (N, M))
    ref = Kx.linear(W, x, bias_bits=b, act="relu", residual_bits=res)
    for h in (0, 1, 16, 63, 64):
        y = Kx.split_linear(W[:h], W[h:], x, bias_bits=b, act="relu", residual_bits=res)
        assert np.array_equal(y, ref)
    t = Kx.bf16_to_f64(x) @ Kx.bf16_to_f64(W).T + Kx.bf16_to_f64(b)
    assert np.allclose(ref, np.maximum(t, 0) + Kx.bf16_to_f64(res), rtol=0, atol=1e-12)


def _make_paged(Ls, Hkv, d, page, host_frac, seed, kind="normal", Hq=None):
    """Logical KV -> two page pools + block table, host = oldest pages (DESIGN reading)."""
    Hq = Hq or Hkv
    q, K, V = synth.kv_inputs(Ls, Hkv, d, Hq, seed, kind=kind)
    g = np.random.default_rng(seed + 1)
    B = len(Ls)
    max_pages = max(-(-L // page) for L in Ls)
    n_host = []
    pages = []
    for b, L in enumerate(Ls):
        npg = -(-L // page)
        nh = int(round(host_frac * npg))
        n_host.append(nh)
        pages.append(npg)
    Ph, Pg = sum(n_host), sum(p - h for p, h in zip(pages, n_host))
    kh = np.zeros((max(Ph, 1), Hkv, page, d), np.uint16)
    vh = np.zeros_like(kh)
    kg = np.zeros((max(Pg, 1), Hkv, page, d), np.uint16)
    vg = np.zeros_like(kg)
    bt = np.zeros((B, max_pages), np.int64)
    ih = list(g.permutation(max(Ph, 1)))
    ig = list(g.permutation(max(Pg, 1)))
    for b, L in enumerate(Ls):
        for p in range(pages[b]):
            tok = slice(p * page, min(L, (p + 1) * page))
            n = tok.stop - tok.start
            if p < n_host[b]:
                j = int(ih.pop())
                kh[j, :, :n] = K[b][tok].transpose(1, 0, 2)
                vh[j, :, :n] = V[b][tok].transpose(1, 0, 2)
                bt[b, p] = j | 0x80000000
            else:
                j = int(ig.pop())
                kg[j, :, :n] = K[b][tok].transpose(1, 0, 2)
                vg[j, :, :n] = V[b][tok].transpose(1, 0, 2)
                bt[b, p] = j
    bt = bt.astype(np.uint32).view(np.int32) if False else (bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    return q, K, V, (kg, vg, kh, vh, bt)


def test_paged_attention_equals_dense_and_tier_invariance():
    Ls = [1, 37, 130, 64]
    q, K, V, (kg, vg, kh, vh, bt) = _make_paged(Ls, 2, 64, 16, 0.5, seed=77, Hq=8)
    o = Kx.paged_attention(q, kg, vg, kh, vh, bt, Ls, 16)
    o2 = Kx.attention_dense(q, K, V)
    assert np.allclose(o, o2, rtol=1e-13, atol=1e-14)
    _, _, _, (kg0, vg0, kh0, vh0, bt0) = _make_paged(Ls, 2, 64, 16, 0.0, seed=77, Hq=8)
    o0 = Kx.paged_attention(q, kg0, vg0, kh0, vh0, bt0, Ls, 16)
    assert np.allclose(o, o0, rtol=1e-13, atol=1e-14)


def test_attention_special_cases():
    d = 32
    # seq_len = 1 -> o = V_0
    q, K, V, (kg, vg, kh, vh, bt) = _make_paged([1, 1], 1, d, 8, 0.0, seed=5, Hq=4)
    o = Kx.paged_attention(q, kg, vg, kh, vh, bt, [1, 1], 8)
    for b in range(2):
        for h in range(4):
            assert np.array_equal(o[b, h], Kx.bf16_to_f64(V[b][0, 0]))
    # constant K -> mean of V
    L = 23
    q, K, V = synth.kv_inputs([L], 1, d, 1, seed=9)
    K[0][:] = K[0][0:1]
    o = Kx.attention_dense(q, K, V)
    assert np.allclose(o[0, 0], Kx.bf16_to_f64(V[0][:, 0]).mean(axis=0), rtol=1e-12, atol=1e-12)
    # one dominant score -> V at the argmax
    K[0][:] = synth.bf16_bits(np.zeros((L, 1, d), np.float32))
    K[0][11, 0, :] = synth.bf16_bits(np.full(d, 64.0, np.float32))
    q[0, 0, :] = synth.bf16_bits(np.full(d, 64.0, np.float32))
    o = Kx.attention_dense(q, K, V)
    assert np.allclose(o[0, 0], Kx.bf16_to_f64(V[0][11, 0]), atol=1e-12)


def test_attention_vs_torch_sdpa_float64():
    torch = pytest.importorskip("torch")
    Ls = [70, 129]
    Hkv, Hq, d = 2, 8, 64
    q, K, V, (kg, vg, kh, vh, bt) = _make_paged(Ls, Hkv, d, 16, 0.25, seed=21, Hq=Hq)
    o = Kx.paged_attention(q, kg, vg, kh, vh, bt, Ls, 16)
    for b, L in enumerate(Ls):
        qq = torch.from_numpy(Kx.bf16_to_f64(q[b])).view(Hq, 1, d)
        kk = torch.from_numpy(Kx.bf16_to_f64(K[b])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0)
        vv = torch.from_numpy(Kx.bf16_to_f64(V[b])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0)
        ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv).view(Hq, d).numpy()
        assert np.allclose(o[b], ref, rtol=1e-12, atol=1e-12)


def test_lse_merge_equals_full_softmax():
    g = np.random.default_rng(1)
    s = g.standard_normal(100)
    V = g.standard_normal((100, 8))
    full = (np.exp(s - s.max()) / np.exp(s - s.max()).sum()) @ V
    cuts = [0, 13, 50, 51, 100]
    os_, ls_ = [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        m = s[a:b].max()
        p = np.exp(s[a:b] - m)
        os_.append(p @ V[a:b] / p.sum())
        ls_.append(m + np.log(p.sum()))
    assert np.allclose(Kx.lse_merge(os_, ls_), full, rtol=1e-13, atol=1e-14)


def test_layernorm_closed_form():
    x = np.array([[1.0, 2.0, 3.0, 4.0]])
    y = Kx.layernorm(x, np.ones(4), np.zeros(4), eps=0.0)
    assert np.allclose(y, (x - 2.5) / np.sqrt(1.25))


def test_rmsnorm_pins():
    """RMSNorm: a constant row c maps to sign(c) * w (eps = 0); invariant to positive scaling;
    equals the Llama reference module (transformers LlamaRMSNorm)."""
    w = np.array([0.5, -1.0, 2.0, 3.0])
    assert np.allclose(Kx.rmsnorm(np.full((1, 4), -3.0), w, eps=0.0), -w)
    g = np.random.default_rng(11)
    x = g.standard_normal((3, 64))
    w = g.standard_normal(64)
    assert np.allclose(Kx.rmsnorm(7.5 * x, w, eps=0.0), Kx.rmsnorm(x, w, eps=0.0), rtol=1e-13)
    import torch
    from transformers.models.llama.modeling_llama import LlamaRMSNorm
    m = LlamaRMSNorm(64, eps=1e-5).double()
    with torch.no_grad():
        m.weight.copy_(torch.from_numpy(w))
        ref = m(torch.from_numpy(x)).numpy()
    # (the module computes its statistics in float32 even for float64 input)
    assert np.allclose(Kx.rmsnorm(x, w, eps=1e-5), ref, rtol=1e-6, atol=1e-7)


def test_bf16_bits_rne_roundtrip():
    """bits -> value -> bits is the identity on finite bf16 patterns; values round to nearest even."""
    g = np.random.default_rng(21)
    bits = synth.bf16_bits(g.standard_normal(5000).astype(np.float32))
    assert np.array_equal(Kx.bf16_bits_rne(Kx.bf16_to_f64(bits)), bits)
    assert Kx.bf16_to_f64(Kx.bf16_bits_rne(np.array([257.0])))[0] == 256.0


def test_round_to_bf16_matches_bit_definition():
    """round_to_bf16 == the RNE bit rounding of the input generator on float32-exact values, and
    is exact on representable values (integers up to 256, powers of two)."""
    g = np.random.default_rng(4)
    v = g.standard_normal(20000).astype(np.float32)
    assert np.array_equal(Kx.round_to_bf16(v.astype(np.float64)), Kx.bf16_to_f64(synth.bf16_bits(v)))
    ints = np.arange(-256, 257, dtype=np.float64)
    assert np.array_equal(Kx.round_to_bf16(ints), ints)
    assert Kx.round_to_bf16(np.array([257.0]))[0] == 256.0  # tie -> even
    assert Kx.round_to_bf16(np.array([259.0]))[0] == 260.0


def _paged_from_logical(K, V, page, Hkv, d, frac, seed):
    """Lay logical per-request K/V out in paged tier pools (host = the oldest pages)."""
    g = np.random.default_rng(seed)
    B = len(K)
    pages = [-(-k.shape[0] // page) for k in K]
    nh = [int(round(frac * p)) for p in pages]
    Ph, Pg = max(1, sum(nh)), max(1, sum(p - h for p, h in zip(pages, nh)))
    kh, vh = np.zeros((Ph, Hkv, page, d), np.uint16), np.zeros((Ph, Hkv, page, d), np.uint16)
    kg, vg = np.zeros((Pg, Hkv, page, d), np.uint16), np.zeros((Pg, Hkv, page, d), np.uint16)
    bt = np.zeros((B, max(pages)), np.int64)
    ih, ig = list(g.permutation(Ph)), list(g.permutation(Pg))
    for b in range(B):
        for p in range(pages[b]):
            lo, hi = p * page, min(K[b].shape[0], (p + 1) * page)
            host = p < nh[b]
            j = int((ih if host else ig).pop())
            (kh if host else kg)[j, :, :hi - lo] = K[b][lo:hi].transpose(1, 0, 2)
            (vh if host else vg)[j, :, :hi - lo] = V[b][lo:hi].transpose(1, 0, 2)
            bt[b, p] = j | (0x80000000 if host else 0)
    return kg, vg, kh, vh, bt.astype(np.uint32).view(np.int32)


def test_prefill_attention_vs_torch_sdpa_causal():
    """Prefill oracle (T new tokens after a prefix) = torch SDPA in float64 with the causal mask
    offset by the prefix (prefix 0: is_causal=True), any tier split; GQA by repeating kv heads."""
    torch = pytest.importorskip("torch")
    import synth
    d, page, Hq, Hkv = 32, 16, 4, 2
    for Ls, T in (([20, 37], 20), ([50, 9], 9), ([70], 33)):
        q, _, _ = synth.kv_inputs([T] * len(Ls), Hkv, d, Hq * T, seed=11 + T)
        q = q.reshape(len(Ls), T, Hq, d)
        _, K, V = synth.kv_inputs(Ls, Hkv, d, Hq, seed=12 + T)
        for frac in (0.0, 0.5, 1.0):
            kg, vg, kh, vh, bt = _paged_from_logical(K, V, page, Hkv, d, frac, 5)
            got = Kx.paged_prefill_attention(q, kg, vg, kh, vh, bt, Ls, page)
            for b, L in enumerate(Ls):
                qt = torch.from_numpy(Kx.bf16_to_f64(q[b])).permute(1, 0, 2)            # [Hq, T, d]
                kt = torch.from_numpy(Kx.bf16_to_f64(K[b])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0)
                vt = torch.from_numpy(Kx.bf16_to_f64(V[b])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0)
                if L == T:
                    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
                else:
                    mask = torch.arange(L)[None, :] <= (L - T + torch.arange(T))[:, None]
                    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask)
                assert np.allclose(got[b], ref.permute(1, 0, 2).numpy(), rtol=1e-12, atol=1e-12)


def test_prefill_attention_last_row_is_decode():
    """The last query of a prefill sees the whole sequence: it equals the decode oracle; T = 1 is
    decode attention exactly."""
    import synth
    d, page, Hq, Hkv, Ls, T = 32, 16, 4, 2, [40, 77], 5
    q, _, _ = synth.kv_inputs([T] * 2, Hkv, d, Hq * T, seed=3)
    q = q.reshape(2, T, Hq, d)
    _, K, V = synth.kv_inputs(Ls, Hkv, d, Hq, seed=4)
    kg, vg, kh, vh, bt = _paged_from_logical(K, V, page, Hkv, d, 0.5, 6)
    pre = Kx.paged_prefill_attention(q, kg, vg, kh, vh, bt, Ls, page)
    dec = Kx.paged_attention(np.ascontiguousarray(q[:, -1]), kg, vg, kh, vh, bt, Ls, page)
    assert np.allclose(pre[:, -1], dec, rtol=1e-13, atol=1e-13)
