"""GPU parity of dak_attention (split paged GQA decode attention) vs the CPU oracle."""
import numpy as np
import pytest

from oracle import kernels as Kx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2604_26074_b200 import dak
    return dak


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def run_attn(D, torch, Ls, Hkv, Hq, page, chunk_pages, frac, seed, paper_mode=False, kind="normal", **cfg):
    from tests.gpu_util import make_paged_kv, PagedKV, to_dev, from_dev
    d = 128
    q, K, V, (kg, vg, kh, vh, bt), n_host = make_paged_kv(Ls, Hkv, d, page, frac, chunk_pages, seed, Hq,
                                                         kind=kind, paper_mode=paper_mode)
    kv = PagedKV(D, kg, vg, kh, vh, bt, page)
    B = len(Ls)
    qd = to_dev(q)
    out = torch.empty((B, Hq, d), dtype=torch.int16, device="cuda")
    sl = torch.tensor(Ls, dtype=torch.int32, device="cuda")
    a = D.attention_args(qd, out, kv.kg, kv.vg, kv.kh.dp, kv.vh.dp, kv.bt, sl, B, Hq, Hkv, d, page, bt.shape[1],
                         chunk_pages, cfg=cfg)
    ws_bytes = D.attention_workspace_size(a)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws_bytes
    D.attention(a)
    torch.cuda.synchronize()
    ref = Kx.paged_attention(q, kg, vg, kh, vh, bt, Ls, page)
    return from_dev(out), ref, n_host


CASES = [  # (seq lens, Hkv, Hq, page, chunk_pages, host fraction)
    ([1, 100, 700], 2, 8, 64, 4, 0.5),
    ([64, 65, 129, 1], 4, 4, 64, 1, 0.25),      # MHA (OPT-style), ragged last pages
    ([3000, 17], 1, 8, 64, 2, 0.3),             # Llama-70B TP8 shard: 1 kv head x 8 q heads
    ([513], 8, 64, 64, 2, 1.0),                 # all on host
    ([200, 300], 2, 16, 32, 3, 0.0),            # page 32, all HBM
    ([1024, 999], 2, 4, 128, 2, 0.5),           # page 128
]


@pytest.mark.parametrize("Ls,Hkv,Hq,page,cp,frac", CASES)
def test_attention_parity(D, torch, Ls, Hkv, Hq, page, cp, frac):
    from tests.gpu_util import assert_close
    got, ref, _ = run_attn(D, torch, Ls, Hkv, Hq, page, cp, frac, seed=900 + sum(Ls))
    assert_close(Kx.bf16_to_f64(got), ref)


def test_attention_paper_mode_batch_split(D, torch):
    """Paper mode: whole requests in host memory, the rest in HBM."""
    from tests.gpu_util import assert_close
    got, ref, n_host = run_attn(D, torch, [300, 301, 302, 303], 2, 8, 64, 2, 0.5, seed=31, paper_mode=True)
    assert n_host[0] > 0 and n_host[-1] == 0
    assert_close(Kx.bf16_to_f64(got), ref)


def test_attention_r_invariance_bitwise(D, torch):
    """Same logical KV placed with 0%, 50%, 100% of chunks on the host -> bitwise-equal output."""
    outs = []
    for frac in (0.0, 0.5, 1.0):
        got, ref, _ = run_attn(D, torch, [777, 1500], 2, 16, 64, 2, frac, seed=44)
        outs.append(got)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("nh,win,st,cc", [(1, 1, 0, 1), (2, 2, 0, 1), (3, 4, 0, 1), (2, 0, 1, 1), (2, 0, 3, 0),
                                         (16, 0, 0, 1), (1, 0, 16, 0)])
def test_attention_launch_config_invariance(D, torch, nh, win, st, cc):
    """Congestion-control / ring knobs (host CTAs, window, ring-slot cap per warp, congestion cap)
    never change results (bitwise): every unit's reduction order is fixed by the chunking."""
    base, _, _ = run_attn(D, torch, [900, 40], 2, 8, 64, 2, 0.5, seed=55)
    got, _, _ = run_attn(D, torch, [900, 40], 2, 8, 64, 2, 0.5, seed=55, n_cta_host=nh, window=win, n_cta_hbm=37,
                         stages=st, congestion_control=cc)
    assert np.array_equal(base, got)


def test_attention_special_cases(D, torch):
    """seq_len = 1 -> o = V_0 exactly (bf16 in, single weight 1)."""
    got, ref, _ = run_attn(D, torch, [1, 1, 1], 2, 8, 64, 1, 0.5, seed=66)
    assert np.array_equal(Kx.bf16_to_f64(got), ref)


def test_kv_append(D, torch):
    """dak_kv_append writes each request's new token at positions[b] in the named tier."""
    from tests.gpu_util import make_paged_kv, PagedKV, to_dev, from_dev, assert_close
    import synth
    Ls = [130, 64, 1]
    Hkv, Hq, page, d = 2, 8, 64, 128
    q, K, V, (kg, vg, kh, vh, bt), _ = make_paged_kv([L + 1 for L in Ls], Hkv, d, page, 0.5, 1, 77, Hq)
    # blank the last token in the logical pools, then append it through the library
    kg2, vg2, kh2, vh2 = kg.copy(), vg.copy(), kh.copy(), vh.copy()
    for b, L in enumerate(Ls):
        e = int(np.uint32(bt[b, L // page]))
        pool_k, pool_v = (kh2, vh2) if e & 0x80000000 else (kg2, vg2)
        pool_k[e & 0x7FFFFFFF, :, L % page] = 0
        pool_v[e & 0x7FFFFFFF, :, L % page] = 0
    kv = PagedKV(D, kg2, vg2, kh2, vh2, bt, page)
    full = PagedKV(D, kg, vg, kh, vh, bt, page)  # the pools as they must look after the append
    k_new = np.stack([K[b][L] for b, L in enumerate(Ls)])
    v_new = np.stack([V[b][L] for b, L in enumerate(Ls)])
    pos = torch.tensor(Ls, dtype=torch.int32, device="cuda")
    kd, vd = to_dev(k_new), to_dev(v_new)
    D.kv_append(kd, vd, kv.bt, pos, len(Ls), Hkv, d, page, bt.shape[1], kv.kg, kv.vg, kv.kh.dp, kv.vh.dp)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(kv.kg), from_dev(full.kg)) and np.array_equal(from_dev(kv.vg), from_dev(full.vg))
    assert np.array_equal(kv.kh.numpy(), full.kh.numpy()) and np.array_equal(kv.vh.numpy(), full.vh.numpy())
    B = len(Ls)
    out = torch.empty((B, Hq, d), dtype=torch.int16, device="cuda")
    sl = torch.tensor([L + 1 for L in Ls], dtype=torch.int32, device="cuda")
    qd = to_dev(q)  # keep a reference: the workspace allocated below must not reuse q's memory
    a = D.attention_args(qd, out, kv.kg, kv.vg, kv.kh.dp, kv.vh.dp, kv.bt, sl, B, Hq, Hkv, d, page,
                         bt.shape[1], 1)
    ws = torch.zeros(D.attention_workspace_size(a), dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    D.attention(a)
    torch.cuda.synchronize()
    ref = Kx.paged_attention(q, kg, vg, kh, vh, bt, [L + 1 for L in Ls], page)
    assert_close(Kx.bf16_to_f64(from_dev(out)), ref)


@pytest.mark.parametrize("Ls,cp", [([130, 64, 1], 1), ([700, 63, 129], 2), ([2, 1025], 4)])
def test_attention_fused_kv_append(D, torch, Ls, cp):
    """dak_attention with k_new / v_new (the KV append fused into the attention kernel): the pools
    end up exactly as after dak_kv_append (both tiers), and the output equals the oracle over the
    full context (the new token's row is used although the pool row was blank when the kernel
    started). Half of each request's chunks on the host."""
    from tests.gpu_util import make_paged_kv, PagedKV, to_dev, from_dev, assert_close
    Hkv, Hq, page, d = 2, 8, 64, 128
    q, K, V, (kg, vg, kh, vh, bt), _ = make_paged_kv([L + 1 for L in Ls], Hkv, d, page, 0.5, cp, 91, Hq)
    kg2, vg2, kh2, vh2 = kg.copy(), vg.copy(), kh.copy(), vh.copy()
    for b, L in enumerate(Ls):
        e = int(np.uint32(bt[b, L // page]))
        pool_k, pool_v = (kh2, vh2) if e & 0x80000000 else (kg2, vg2)
        pool_k[e & 0x7FFFFFFF, :, L % page] = 0
        pool_v[e & 0x7FFFFFFF, :, L % page] = 0
    kv = PagedKV(D, kg2, vg2, kh2, vh2, bt, page)
    full = PagedKV(D, kg, vg, kh, vh, bt, page)
    # new rows inside a strided [B, (Hq + 2 Hkv) d] buffer, as the fused QKV projection leaves them
    B = len(Ls)
    qkv = np.zeros((B, (Hq + 2 * Hkv) * d), np.uint16)
    qkv[:, Hq * d:(Hq + Hkv) * d] = np.stack([K[b][L] for b, L in enumerate(Ls)]).reshape(B, -1)
    qkv[:, (Hq + Hkv) * d:] = np.stack([V[b][L] for b, L in enumerate(Ls)]).reshape(B, -1)
    qkvd = to_dev(qkv)
    out = torch.empty((B, Hq, d), dtype=torch.int16, device="cuda")
    sl = torch.tensor([L + 1 for L in Ls], dtype=torch.int32, device="cuda")
    qd = to_dev(q)
    a = D.attention_args(qd, out, kv.kg, kv.vg, kv.kh.dp, kv.vh.dp, kv.bt, sl, B, Hq, Hkv, d, page, bt.shape[1], cp,
                         k_new=qkvd.data_ptr() + Hq * d * 2, v_new=qkvd.data_ptr() + (Hq + Hkv) * d * 2,
                         kv_new_stride=(Hq + 2 * Hkv) * d)
    ws = torch.zeros(max(D.attention_workspace_size(a), 16), dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    D.attention(a)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(kv.kg), from_dev(full.kg)) and np.array_equal(from_dev(kv.vg), from_dev(full.vg))
    assert np.array_equal(kv.kh.numpy(), full.kh.numpy()) and np.array_equal(kv.vh.numpy(), full.vh.numpy())
    ref = Kx.paged_attention(q, kg, vg, kh, vh, bt, [L + 1 for L in Ls], page)
    assert_close(Kx.bf16_to_f64(from_dev(out)), ref)
    # and bitwise equal to the unfused path (append first, then attention over the full pools)
    out2 = torch.empty_like(out)
    a2 = D.attention_args(qd, out2, full.kg, full.vg, full.kh.dp, full.vh.dp, full.bt, sl, B, Hq, Hkv, d, page,
                          bt.shape[1], cp, workspace=ws, workspace_bytes=ws.numel())
    D.attention(a2)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(out), from_dev(out2))


@pytest.mark.slow
def test_c4_128k_half_host_sampled(D, torch):
    """BASELINE configs[3]: GQA decode attention over a 128k-token context, 64 q / 8 kv heads,
    50% of the KV (oldest chunks) in host memory; full output vs the oracle."""
    from tests.gpu_util import assert_close
    got, ref, n_host = run_attn(D, torch, [131072], 8, 64, 64, 16, 0.5, seed=0xDA0 + 3)
    assert n_host[0] == 1024
    assert_close(Kx.bf16_to_f64(got), ref)


def test_attention_errors(D, torch):
    a = D.attention_args(16, 16, 16, 16, None, None, 16, 16, 1, 6, 4, 128, 64, 4, 1, cfg=dict(n_cta_hbm=4))
    with pytest.raises(D.DakError):
        D.attention_workspace_size(a)  # Hq % Hkv != 0
    a = D.attention_args(16, 16, 16, 16, None, None, 16, 16, 1, 8, 8, 64, 64, 4, 1, cfg=dict(n_cta_hbm=4))
    with pytest.raises(D.DakError) as e:
        D.attention_workspace_size(a)  # d != 128
    assert e.value.code == "EUNSUPPORTED"


def test_attention_few_keys_cancellation(D, torch):
    """Two to five keys: o is a weighted mean of a few V rows that often cancels to |o| << |V|, so
    the weights' rounding shows directly (P is fp16 for the P V product: per-element tolerance
    holds; with bf16 weights such rows missed 1e-2 by ~1.6x)."""
    from tests.gpu_util import assert_close
    got, ref, _ = run_attn(D, torch, [2, 3, 4, 5] * 4, 2, 16, 64, 1, 0.5, seed=123)
    assert_close(Kx.bf16_to_f64(got), ref)
