"""GPU parity of the fused pre-norm linear (dak_linear_args.ln_*) and of the epilogue row
statistics (stats_out) against the CPU oracle: LN(x) (or RMSNorm) rounded to bf16, then the
split GEMV (PAPER §3.1 operator; OPT pre-LayerNorm P:L690, Llama RMSNorm for BASELINE C3).

The statistics the fused linear merges come either from dak_row_stats (one part per row) or from
the stats_out epilogue of a producing dak_linear (one part per CTA): both must give LN(x).
"""
import numpy as np
import pytest

import synth
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


def _norm_inputs(K, N, seed, rms=False):
    g = synth.rng(seed)
    x = synth.bf16_bits((g.standard_normal((N, K)) * 2.0 + 0.7).astype(np.float32))  # offset mean
    w = synth.bf16_bits((1.0 + 0.3 * g.standard_normal(K)).astype(np.float32))
    b = None if rms else synth.bf16_bits((0.2 * g.standard_normal(K)).astype(np.float32))
    return x, w, b


def _oracle_norm(x, w, b, rms, eps=1e-5):
    xf = Kx.bf16_to_f64(x)
    if rms:
        h = Kx.rmsnorm(xf, Kx.bf16_to_f64(w), eps)
    else:
        h = Kx.layernorm(xf, Kx.bf16_to_f64(w), Kx.bf16_to_f64(b), eps)
    return Kx.round_to_bf16(h)


@pytest.mark.parametrize("rms", [False, True])
@pytest.mark.parametrize("M,K,N,h,kc", [(700, 1024, 1, 33, 128), (1500, 2048, 8, 64, 256), (512, 4096, 16, 0, 64),
                                        (333, 512, 5, 333, 64), (1024, 8192, 64, 32, 256), (900, 2048, 40, 0, 128)])
def test_fused_norm_linear(D, torch, rms, M, K, N, h, kc):
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    W, _, bias = synth.linear_inputs(M, K, N, seed=synth.seed_for(5, M + N), bias=True)
    x, w, b = _norm_inputs(K, N, seed=M * 7 + N, rms=rms)
    sl = SplitLinear(D, W, h, kc)
    xd, wd = to_dev(x), to_dev(w)
    bd = to_dev(b) if b is not None else None
    stats = torch.zeros((N, 4), dtype=torch.float32, device="cuda")
    D.row_stats(xd, N, K, stats)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    biasd = to_dev(bias)  # keep every device buffer referenced until the kernels ran
    a = sl.args(xd, y, N, bias=biasd)
    a.ln_w, a.ln_b, a.ln_stats = wd.data_ptr(), (bd.data_ptr() if bd is not None else None), stats.data_ptr()
    a.ln_parts, a.ln_rms, a.ln_eps = 1, int(rms), 1e-5
    D.linear(a)
    torch.cuda.synchronize()
    hx = _oracle_norm(x, w, b, rms)
    ref = Kx.split_linear(W[:h], W[h:], synth.bf16_bits(hx.astype(np.float32)), bias_bits=bias)
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("M,N,h,path", [(7168, 8, 56, 0), (1024, 3, 0, 0), (320, 16, 320, 0), (7168, 64, 64, 3),
                                         (2048, 40, 0, 3)])
def test_stats_epilogue_then_fused_norm(D, torch, M, N, h, path):
    """Producer linear writes per-CTA (count, mean, M2) of its bf16 outputs; (1) the merged
    statistics equal mean / variance of those outputs, (2) a consumer linear fused with LN over
    them equals LN(y) -> GEMV in the oracle."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    K = 1024
    W, x, bias = synth.linear_inputs(M, K, N, seed=synth.seed_for(6, M), bias=True)
    sl = SplitLinear(D, W, h, 64 if path == 3 else 128)
    xd = to_dev(x)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    biasd = to_dev(bias)  # keep every device buffer referenced until the kernels ran
    a = sl.args(xd, y, N, bias=biasd, force_path=path)
    grid = D.linear_query(a)["grid"]
    stats = torch.full((grid, N, 4), float("nan"), dtype=torch.float32, device="cuda")
    a.stats_out = stats.data_ptr()
    D.linear(a)
    torch.cuda.synchronize()
    yb = from_dev(y)
    yf = Kx.bf16_to_f64(yb)
    st = stats.cpu().numpy().astype(np.float64)
    cnt = st[:, :, 0].sum(axis=0)
    assert np.array_equal(cnt, np.full(N, M))
    mean = (st[:, :, 0] * st[:, :, 1]).sum(axis=0) / cnt
    m2 = st[:, :, 2].sum(axis=0) + (st[:, :, 0] * (st[:, :, 1] - mean) ** 2).sum(axis=0)
    assert np.allclose(mean, yf.mean(axis=1), rtol=1e-4, atol=1e-5)
    assert np.allclose(m2 / M, yf.var(axis=1), rtol=1e-4)
    # consumer: LN fused over the producer's partials
    M2_, h2 = 640, 40
    W2, _, b2 = synth.linear_inputs(M2_, M, N, seed=synth.seed_for(7, M), bias=True)
    _, w, b = _norm_inputs(M, 1, seed=3)
    sl2 = SplitLinear(D, W2, h2, 128 if M % 128 == 0 else 64)
    z = torch.empty((N, M2_), dtype=torch.int16, device="cuda")
    b2d = to_dev(b2)
    a2 = sl2.args(y, z, N, bias=b2d)
    wd, bd = to_dev(w), to_dev(b)
    a2.ln_w, a2.ln_b, a2.ln_stats, a2.ln_parts, a2.ln_eps = wd.data_ptr(), bd.data_ptr(), stats.data_ptr(), grid, 1e-5
    D.linear(a2)
    torch.cuda.synchronize()
    hy = _oracle_norm(yb, w, b, rms=False)
    ref = Kx.split_linear(W2[:h2], W2[h2:], synth.bf16_bits(hy.astype(np.float32)), bias_bits=b2)
    assert_close(Kx.bf16_to_f64(from_dev(z)), ref)


def test_embed_stats(D, torch):
    from tests.gpu_util import to_dev, from_dev
    g = synth.rng(9)
    V, H, B = 100, 7168, 4
    te = synth.bf16_bits(g.standard_normal((V, H)).astype(np.float32))
    pe = synth.bf16_bits(g.standard_normal((20, H)).astype(np.float32))
    tok = torch.tensor([3, 99, 0, 3], dtype=torch.int32, device="cuda")
    pos = torch.tensor([0, 5, 17, 2], dtype=torch.int32, device="cuda")
    x = torch.empty((B, H), dtype=torch.int16, device="cuda")
    stats = torch.zeros((B, 4), dtype=torch.float32, device="cuda")
    D.embed(tok, pos, to_dev(te), to_dev(pe), B, H, 2, x, stats_out=stats)
    torch.cuda.synchronize()
    ref = Kx.round_to_bf16(Kx.bf16_to_f64(te)[tok.cpu().numpy()] + Kx.bf16_to_f64(pe)[pos.cpu().numpy() + 2])
    xf = Kx.bf16_to_f64(from_dev(x))
    assert np.array_equal(xf, ref)
    st = stats.cpu().numpy()
    assert np.array_equal(st[:, 0], np.full(B, H))
    assert np.allclose(st[:, 1], xf.mean(axis=1), rtol=1e-4, atol=1e-6)
    assert np.allclose(st[:, 2] / H, xf.var(axis=1), rtol=1e-4)
