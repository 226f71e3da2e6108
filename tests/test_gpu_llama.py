"""GPU parity of the Llama decode step (DakLlama: dak_layer DAK_MODEL_LLAMA through the C ABI)
against the CPU oracle (oracle/layer.py llama_decode_step, pinned to transformers Llama), with
weights and KV split between HBM and pinned host memory, and with the row-parallel combine going
through an NCCL communicator (1 rank on one GPU: the all-reduce path runs, the sum is identity)."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly

pytestmark = pytest.mark.gpu


def _dev(p, torch):
    return {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16)).cuda().view(torch.bfloat16) for k, v in p.items()}


@pytest.mark.parametrize("frac,B,ctx,use_comm,fuse", [(0.0, 3, 70, False, True), (0.3, 2, 150, False, True),
                                                     (0.2, 4, 40, True, True), (0.2, 4, 40, True, False),
                                                     (0.3, 24, 90, False, None), (0.3, 24, 90, True, None),
                                                     (0.0, 300, 70, True, None)])  # B > 256: CTA-pair linears
def test_llama_step_matches_oracle(frac, B, ctx, use_comm, fuse):
    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import HW
    from paper_2604_26074_b200.llama import DakLlama, LlamaConfig
    from tests.test_oracle_llama import make_llama_params
    L, H, F, V, nh, nkv, d = 2, 512, 768, 96, 4, 2, 128
    g = synth.rng(4242)
    p = make_llama_params(g, L, H, F, V, nh, nkv, d)
    cfg = LlamaConfig(n_layers=L, hidden=H, n_heads=nh, n_kv_heads=nkv, ffn=F, vocab=V, name="llama-tiny")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    comm = dak.comm_init(dak.comm_unique_id(), 0, 1) if use_comm else None
    total = L * (H * (nh + 2 * nkv) * d + nh * d * H + 3 * F * H) * 2 + V * H * 2
    eng = DakLlama(cfg, B, ctx, hw, comm=comm, mode=dak.PLAN_EXACT, y_req=int(frac * total), page_size=64,
                   chunk_pages=1, weights=_dev(p, torch), fuse_norm=fuse)
    if frac > 0:
        assert sum(op.h for op in eng.linear_ops()) > 0
    Kc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    tokens = (np.arange(B) * 13 + 3) % V
    eng.tokens.copy_(torch.from_numpy(tokens.astype(np.int32)))
    s = torch.cuda.Stream()
    eng.capture(s)
    eng.graph.replay()
    torch.cuda.synchronize()
    ref, _ = Ly.llama_decode_step(tokens, np.full(B, ctx - 1), p, Kc, Vc, nh, nkv)
    got = Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16))
    from tests.gpu_util import assert_close
    assert_close(got, ref, rtol=3e-2)
    eng.close()
    if comm:
        dak.comm_destroy(comm)


def test_rope_kv_append_matches_oracle():
    """Rotated q (in place) and the rotated k / v rows written into the paged pools."""
    import torch
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import to_dev, from_dev
    B, Hq, Hkv, d, page, max_pages = 3, 8, 2, 128, 64, 4
    g = synth.rng(99)
    qkv = synth.normal_bf16(g, (B, (Hq + 2 * Hkv) * d), 1.0)
    pos = np.array([0, 77, 250], dtype=np.int32)
    bt = np.array([[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 0x80000000 | 0]], dtype=np.int64)
    bt32 = torch.from_numpy((bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda()
    qd = to_dev(qkv)
    kg = torch.zeros(12 * Hkv * page * d, dtype=torch.int16, device="cuda")
    vg = torch.zeros_like(kg)
    from tests.gpu_util import HostBuf
    kh, vh = HostBuf(dak, Hkv * page * d * 2), HostBuf(dak, Hkv * page * d * 2)
    dak.rope_kv_append(qd, 0, B, Hq, Hkv, d, torch.from_numpy(pos).cuda(), 500000.0, bt32, page, max_pages, kg, vg,
                       kh.dp, vh.dp)
    torch.cuda.synchronize()
    out = Kx.bf16_to_f64(from_dev(qd)).reshape(B, Hq + 2 * Hkv, d)
    x = Kx.bf16_to_f64(qkv).reshape(B, Hq + 2 * Hkv, d)
    for b in range(B):
        ref_q = Kx.round_to_bf16(Ly.rope(x[b, :Hq], int(pos[b]), 500000.0))
        ref_k = Kx.round_to_bf16(Ly.rope(x[b, Hq:Hq + Hkv], int(pos[b]), 500000.0))
        from tests.gpu_util import assert_bf16_ulps
        assert_bf16_ulps(out[b, :Hq], ref_q, ulps=1, floor=1e-6)
        assert_bf16_ulps(out[b, Hq:Hq + Hkv], ref_k, ulps=1, floor=1e-6)
        # pool rows (DAK-PG swizzle): un-swizzle the written row and compare with the rotated k / v
        e = int(bt[b, pos[b] // page])
        t = int(pos[b]) % page
        for pool_k, pool_v in ((kg.cpu().numpy().view(np.uint16), vg.cpu().numpy().view(np.uint16)),):
            pass
        if e & 0x80000000:
            kp, vp = kh.numpy(), vh.numpy()
        else:
            kp, vp = kg.cpu().numpy().view(np.uint16), vg.cpu().numpy().view(np.uint16)
        idx = e & 0x7FFFFFFF
        for gkv in range(Hkv):
            base = (idx * Hkv + gkv) * page * d
            row = np.zeros(d, np.uint16)
            rowv = np.zeros(d, np.uint16)
            for j in range(d // 8):
                c = ((j >> 3) << 3) | ((j & 7) ^ (t & 7))
                row[j * 8:(j + 1) * 8] = kp[base + t * d + c * 8: base + t * d + c * 8 + 8]
                rowv[j * 8:(j + 1) * 8] = vp[base + t * d + c * 8: base + t * d + c * 8 + 8]
            assert np.array_equal(row, from_dev(qd).reshape(B, Hq + 2 * Hkv, d)[b, Hq + gkv])
            assert np.array_equal(rowv, qkv.reshape(B, Hq + 2 * Hkv, d)[b, Hq + Hkv + gkv])


@pytest.mark.parametrize("L,use_comm", [(1, False), (2, True)])
def test_llama_tp8_shard_shapes_b64(L, use_comm):
    """Llama-3-70B layers at the per-GPU shapes of TP8 (hidden 8192, 8 q heads / 1 kv head, FFN 3584,
    batch 64 -> N = 64 GEMV columns, GQA group 8), host share forced, vs the oracle. With a one-rank
    communicator (the bench's path) the o / down split-K partials are reduced inside the residual +
    RMSNorm combine kernel (no reduce launch)."""
    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import HW
    from paper_2604_26074_b200.llama import DakLlama, LlamaConfig
    from tests.test_oracle_llama import make_llama_params
    H, F, V, nh, nkv, d, B, ctx = 8192, 3584, 256, 8, 1, 128, 64, 80
    g = synth.rng(7070)
    p = make_llama_params(g, L, H, F, V, nh, nkv, d)
    cfg = LlamaConfig(n_layers=L, hidden=H, n_heads=nh, n_kv_heads=nkv, ffn=F, vocab=V, name="llama-tp8-shard")
    hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
    total = (H * (nh + 2 * nkv) * d + nh * d * H + 3 * F * H) * 2 + V * H * 2
    comm = dak.comm_init(dak.comm_unique_id(), 0, 1) if use_comm else None
    eng = DakLlama(cfg, B, ctx, hw, mode=dak.PLAN_EXACT, y_req=int(0.05 * L * total), page_size=64, chunk_pages=1,
                   weights=_dev(p, torch), comm=comm)
    assert sum(op.h for op in eng.linear_ops()) > 0
    Kc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    tokens = (np.arange(B) * 7) % V
    eng.tokens.copy_(torch.from_numpy(tokens.astype(np.int32)))
    s = torch.cuda.Stream()
    eng.capture(s)
    eng.graph.replay()
    torch.cuda.synchronize()
    ref, _ = Ly.llama_decode_step(tokens, np.full(B, ctx - 1), p, Kc, Vc, nh, nkv)
    got = Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16))
    from tests.gpu_util import assert_close
    assert_close(got, ref, rtol=3e-2)
    eng.close()
    if comm:
        dak.comm_destroy(comm)


def test_rmsnorm_and_silu_mul_kernels():
    import torch
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import to_dev, from_dev
    g = synth.rng(31)
    x = synth.normal_bf16(g, (5, 8192), 1.3)
    w = synth.bf16_bits((1.0 + 0.2 * g.standard_normal(8192)).astype(np.float32))
    y = torch.empty((5, 8192), dtype=torch.int16, device="cuda")
    xd, wd = to_dev(x), to_dev(w)
    dak.rmsnorm(xd, wd, y, 5, 8192, 1e-5)
    gu = synth.normal_bf16(g, (3, 2 * 3584), 2.0)
    gd = to_dev(gu)
    o = torch.empty((3, 3584), dtype=torch.int16, device="cuda")
    dak.silu_mul(gd, o, 3, 3584)
    torch.cuda.synchronize()
    ref = Kx.round_to_bf16(Kx.rmsnorm(Kx.bf16_to_f64(x), Kx.bf16_to_f64(w), 1e-5))
    got = Kx.bf16_to_f64(from_dev(y))
    from tests.gpu_util import assert_bf16_ulps
    assert_bf16_ulps(got, ref)
    gf, uf = Kx.bf16_to_f64(gu[:, :3584]), Kx.bf16_to_f64(gu[:, 3584:])
    ref2 = Kx.round_to_bf16(Ly.silu(gf) * uf)
    got2 = Kx.bf16_to_f64(from_dev(o))
    assert_bf16_ulps(got2, ref2, floor=1e-6)


@pytest.mark.parametrize("rows,cols", [(4, 8192), (3, 520), (2, 16384), (2, 64), (3, 2056), (3, 5000), (2, 6152),
                                       (2, 28672), (1, 65536), (1, 131072)])
def test_allreduce_residual_rmsnorm_kernel(rows, cols):
    """x += partial (bf16 RNE) and y = RMSNorm(x) * w in one kernel (1-rank: no exchange), vs the
    oracle's residual add + rmsnorm; y aliasing partial (as in the Llama layer) gives the same.
    The column counts cover every launch shape of the kernel: 1, 2, 3, 4 and 8 CTAs per row (a
    cluster exchanging the row's sum of squares) and 1, 2, 4 and 8 chunks of 8 columns per thread."""
    import torch
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import to_dev, from_dev
    g = synth.rng(77 + cols)
    x = synth.normal_bf16(g, (rows, cols), 1.1)
    pa = synth.normal_bf16(g, (rows, cols), 0.7)
    w = synth.bf16_bits((1.0 + 0.2 * g.standard_normal(cols)).astype(np.float32))
    xs = Kx.round_to_bf16(Kx.bf16_to_f64(x) + Kx.bf16_to_f64(pa))
    ref = Kx.round_to_bf16(Kx.rmsnorm(xs, Kx.bf16_to_f64(w), 1e-5))
    for alias in (False, True):
        xd, pd, wd = to_dev(x), to_dev(pa), to_dev(w)
        y = pd if alias else torch.empty((rows, cols), dtype=torch.int16, device="cuda")
        dak.allreduce_residual_rmsnorm(None, pd, xd, rows, cols, wd, 1e-5, y)
        torch.cuda.synchronize()
        assert np.array_equal(Kx.bf16_to_f64(from_dev(xd)), xs)  # bf16(x + p): exact
        got = Kx.bf16_to_f64(from_dev(y))
        from tests.gpu_util import assert_bf16_ulps
        assert_bf16_ulps(got, ref)


@pytest.mark.parametrize("cols,bias", [(8192, True), (8192, False), (7168, True), (1000, True)])
def test_layernorm_vectorised_and_scalar(cols, bias):
    """dak_layernorm on the vectorised path (cols % 8 == 0) and the scalar fallback (cols = 1000 is
    vectorised too; odd strides are exercised by the OPT engine tests) vs the oracle LayerNorm."""
    import torch
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import to_dev, from_dev
    g = synth.rng(5 + cols)
    x = synth.normal_bf16(g, (6, cols), 1.3)
    w = synth.bf16_bits((1.0 + 0.2 * g.standard_normal(cols)).astype(np.float32))
    b = synth.normal_bf16(g, (cols,), 0.1) if bias else None
    y = torch.empty((6, cols), dtype=torch.int16, device="cuda")
    dak.layernorm(to_dev(x), to_dev(w), to_dev(b) if bias else None, y, 6, cols, 1e-5)
    torch.cuda.synchronize()
    ref = Kx.round_to_bf16(Kx.layernorm(Kx.bf16_to_f64(x), Kx.bf16_to_f64(w),
                                        Kx.bf16_to_f64(b) if bias else np.zeros(cols), 1e-5))
    got = Kx.bf16_to_f64(from_dev(y))
    from tests.gpu_util import assert_bf16_ulps
    assert_bf16_ulps(got, ref)


@pytest.mark.parametrize("rows,cols", [(3, 8192), (2, 1000), (4, 520), (3, 1001), (2, 77)])
def test_allreduce_residual_stats_kernel(rows, cols):
    """x += partial (bf16 RNE) and per-row (cols, mean, M2) of the new x (1-rank: no exchange) vs
    the oracle (float64 statistics of the bf16 row). cols % 8 == 0 takes the vectorised kernel,
    cols = 1001 / 77 the scalar one (the two sum the row in different orders: the statistics agree
    with the oracle within fp32 rounding, not bitwise with each other)."""
    import torch
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import to_dev, from_dev
    g = synth.rng(303 + cols)
    x = synth.normal_bf16(g, (rows, cols), 1.1)
    pa = synth.normal_bf16(g, (rows, cols), 0.7)
    xs = Kx.round_to_bf16(Kx.bf16_to_f64(x) + Kx.bf16_to_f64(pa))
    xd, pd = to_dev(x), to_dev(pa)
    st = torch.zeros((rows, 4), dtype=torch.float32, device="cuda")
    dak.allreduce_residual(None, pd, xd, rows, cols, st)
    torch.cuda.synchronize()
    assert np.array_equal(Kx.bf16_to_f64(from_dev(xd)), xs)
    s = st.cpu().numpy().astype(np.float64)
    assert np.array_equal(s[:, 0], np.full(rows, cols))
    mean, m2 = xs.mean(axis=1), ((xs - xs.mean(axis=1, keepdims=True)) ** 2).sum(axis=1)
    assert np.allclose(s[:, 1], mean, atol=1e-5, rtol=1e-5) and np.allclose(s[:, 2], m2, rtol=1e-4)
