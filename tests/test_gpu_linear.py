"""GPU parity of dak_linear (split GEMV / skinny GEMM, PAPER §3.1) against the CPU oracle.

All calls go through the C ABI (libdak.so) via the ctypes binding. Tolerance (north star):
bf16 outputs with fp32 accumulation within 1e-2 relative; integer inputs bit-exact.
"""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import planner as P

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


def run_linear(D, torch, W, x, h, kc, bias=None, residual=None, act=0, **cfg):
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    M, K = W.shape
    N = x.shape[0]
    sl = SplitLinear(D, W, h, kc)
    xd = to_dev(x)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    bd = to_dev(bias) if bias is not None else None
    rd = to_dev(residual) if residual is not None else None
    a = sl.args(xd, y, N, bias=bd, residual=rd, act=act, **cfg)
    D.linear(a)
    torch.cuda.synchronize()
    return from_dev(y), sl, a


CASES = [  # (M, K, N, h, kc) — several tiles, ragged row counts, both tiers, both paths
    (300, 512, 1, 37, 64),
    (1000, 1024, 3, 0, 128),
    (777, 2048, 4, 777, 256),
    (4096, 4096, 1, 32, 512),
    (513, 256, 8, 100, 64),
    (1024, 4096, 16, 48, 256),
    (2000, 1536, 5, 16, 512),
    (129, 8192, 12, 1, 1024),
    (5000, 128, 2, 2500, 64),
    (1024, 8192, 24, 32, 256),   # 4 n8 tiles
    (3584, 8192, 64, 48, 256),   # 8 n8 tiles (Llama-3-70B TP8 gate/up shard, b64)
    (700, 1024, 33, 0, 128),
]


@pytest.mark.parametrize("M,K,N,h,kc", CASES)
def test_linear_parity(D, torch, M, K, N, h, kc):
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, M + N), bias=True)
    y, _, _ = run_linear(D, torch, W, x, h, kc, bias=b)
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y), ref)


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("N", [1, 4])
def test_linear_integer_exact(D, torch, path, N):
    """Integer inputs in [-2, 2]: every partial sum is an exact small integer -> bitwise equal."""
    M, K = 611, 2048
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, 7), kind="int", bias=True)
    y, _, _ = run_linear(D, torch, W, x, 40, 256, bias=b, force_path=path)
    ref = Kx.split_linear(W[:40], W[40:], x, bias_bits=b)
    assert np.all(ref == np.round(ref))  # exact integer accumulation in the oracle
    assert np.array_equal(Kx.bf16_to_f64(y), Kx.round_to_bf16(ref))


@pytest.mark.parametrize("N,kc", [(1, 512), (3, 64), (8, 256), (16, 128)])
def test_linear_r_invariance_bitwise(D, torch, N, kc):
    """Outputs are bitwise identical for every split point h and CTA count (fixed KC)."""
    M, K = 1536, 4096
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, 11))
    outs = []
    for h, nh in ((0, 1), (16, 1), (300, 2), (768, 3), (M, 5)):
        y, _, _ = run_linear(D, torch, W, x, h, kc, n_cta_host=nh)
        outs.append(y)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(outs[0]), Kx.linear(W, x))


def test_linear_epilogue_relu_residual_inplace(D, torch):
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    M, K, N = 1000, 2048, 8
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, 13), bias=True)
    res = synth.normal_bf16(np.random.default_rng(3), (N, M))
    sl = SplitLinear(D, W, 64, 256)
    xd = to_dev(x)
    y = to_dev(res)  # residual aliases y (in-place residual add, decoder layer use)
    D.linear(sl.args(xd, y, N, bias=to_dev(b), residual=y, act=D.ACT_RELU))
    torch.cuda.synchronize()
    ref = Kx.linear(W, x, bias_bits=b, act="relu", residual_bits=res)
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("path", [1, 2])
def test_linear_paths_agree(D, torch, path):
    M, K, N = 2048, 4096, 4
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, 17))
    y, _, _ = run_linear(D, torch, W, x, 32, 512, force_path=path)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y), Kx.linear(W, x))


def test_linear_pdl_chain(D, torch):
    """A chain y1 = W1 x, y2 = W2 y1, y3 = W3 y2 launched with programmatic dependent launch:
    weights stream early, the x read waits for the producer kernel (griddepcontrol.wait)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    K = 2048
    N = 2
    g = np.random.default_rng(5)
    Ws = [synth.normal_bf16(g, (K, K), std=1 / np.sqrt(K)) for _ in range(3)]
    x = synth.normal_bf16(g, (N, K))
    sls = [SplitLinear(D, W, 32 * (i + 1), 256) for i, W in enumerate(Ws)]
    bufs = [to_dev(x)] + [torch.empty((N, K), dtype=torch.int16, device="cuda") for _ in range(3)]
    for rep in range(3):
        for i in range(3):
            D.linear(sls[i].args(bufs[i], bufs[i + 1], N, pdl=1))
    torch.cuda.synchronize()
    ref = x
    for W in Ws:
        r = Kx.linear(W, ref)
        ref = synth.bf16_bits(r.astype(np.float32))  # bf16 RNE between ops (float32 rounding then bf16)
    got = from_dev(bufs[3])
    assert_close(Kx.bf16_to_f64(got), Kx.bf16_to_f64(ref), rtol=2e-2)


def test_c1_full_size_at_planner_ratio(D, torch):
    """BASELINE configs[0]: 4096x4096 bf16 GEMV, N=1, split at the planner's BALANCED ratio
    (unit 16 rows), in the launch configuration bench.py times; full output compared."""
    M = K = 4096
    Bg, Bh = 6555.5e9, 51.5e9
    plan, _ = D.plan_ratios(dict(hbm_bps=Bg, link_bps=Bh, host_dram_bps=Bh),
                            [dict(n_units=M // 16, unit_bytes=16 * K * 2, total_bytes=M * K * 2, T=0.0)], 0,
                            D.PLAN_BALANCED)
    h = plan[0]["host_units"] * 16
    assert 16 <= h <= 64
    W, x, _ = synth.linear_inputs(M, K, 1, seed=synth.seed_for(0, 0))
    kc = D.default_kc(M, K, 147)
    y, sl, a = run_linear(D, torch, W, x, h, kc)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y), Kx.linear(W, x))
    info = D.linear_query(a)
    assert info["n_cta_host"] >= 1 and info["host_bytes"] == h * K * 2


@pytest.mark.parametrize("M,K,N", [(28672, 7168, 8), (7168, 28672, 1), (50272, 7168, 8)])
def test_opt30b_shapes_sampled(D, torch, M, K, N):
    """OPT-30B fc1 / fc2 / LM-head shapes (configs[1]) at r ~ r*: sampled rows vs the row-loop oracle."""
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(1, M % 1000))
    h = 16 * max(1, round(M * 0.0078 / 16))
    y, _, _ = run_linear(D, torch, W, x, h, D.default_kc(M, K, 147))
    rows = np.unique(np.concatenate([np.arange(0, 40), np.arange(h - 8, h + 8),
                                     np.random.default_rng(0).integers(0, M, 200), np.arange(M - 20, M)]))
    ref = Kx.linear_rowloop(W[rows], x)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y[:, rows]), ref)


@pytest.mark.parametrize("M,K,N,h,kc", [(1000, 1024, 8, 24, 128), (3584, 2048, 64, 32, 256), (640, 512, 3, 640, 64)])
def test_linear_swiglu_operand(D, torch, M, K, N, h, kc):
    """x = [gate | up] of width 2K; the GEMV operand is bf16(silu(gate) * up) (Llama MLP down proj)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    W, _, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(8, M + N))
    g = synth.rng(M * 3 + N)
    gu = synth.normal_bf16(g, (N, 2 * K), 1.5)
    sl = SplitLinear(D, W, h, kc)
    xd = to_dev(gu)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    a = sl.args(xd, y, N)
    a.x_swiglu = 1
    D.linear(a)
    torch.cuda.synchronize()
    gf, uf = Kx.bf16_to_f64(gu[:, :K]), Kx.bf16_to_f64(gu[:, K:])
    act = Kx.round_to_bf16(gf / (1.0 + np.exp(-gf)) * uf)
    ref = Kx.split_linear(W[:h], W[h:], synth.bf16_bits(act.astype(np.float32)))
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("M,K,N,h,kc,xf", [(7168, 7168, 8, 48, 256, 0), (3584, 8192, 64, 32, 256, 0),
                                           (1500, 2048, 8, 64, 256, 1), (1000, 1024, 16, 0, 128, 2)])
@pytest.mark.parametrize("cluster", [2, 4])
def test_linear_x_multicast_bitwise(D, torch, M, K, N, h, kc, xf, cluster):
    """TMA multicast of the x chunk within clusters (one fetch per cluster) gives the
    same outputs bitwise as one fetch per CTA (and both match the oracle)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(9, M + N), bias=True)
    g = synth.rng(M + 17 * N)
    if xf == 2:
        x = synth.normal_bf16(g, (N, 2 * K), 1.0)
    sl = SplitLinear(D, W, h, kc)
    xd, bd = to_dev(x), to_dev(b)
    extra = {}
    if xf == 1:
        w_ln = synth.bf16_bits((1.0 + 0.2 * g.standard_normal(K)).astype(np.float32))
        b_ln = synth.normal_bf16(g, (K,), 0.1)
        wd, bld = to_dev(w_ln), to_dev(b_ln)
        stats = torch.zeros((N, 4), dtype=torch.float32, device="cuda")
        D.row_stats(xd, N, K, stats)
    outs = []
    for cl in (1, cluster):
        y = torch.empty((N, M), dtype=torch.int16, device="cuda")
        a = sl.args(xd, y, N, bias=bd, cluster=cl)
        if xf == 1:
            a.ln_w, a.ln_b, a.ln_stats, a.ln_parts, a.ln_eps = wd.data_ptr(), bld.data_ptr(), stats.data_ptr(), 1, 1e-5
        if xf == 2:
            a.x_swiglu = 1
        info = D.linear_query(a)
        assert info["cluster"] == cl
        D.linear(a)
        torch.cuda.synchronize()
        outs.append(from_dev(y))
    assert np.array_equal(outs[0], outs[1])
    if xf == 0:
        ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
        assert_close(Kx.bf16_to_f64(outs[1]), ref)


@pytest.mark.parametrize("M,K,N,h", [(1024, 8192, 64, 32), (3584, 4096, 32, 0), (7168, 7168, 16, 56),
                                     (1000, 2048, 40, 16), (300, 1024, 64, 296), (28672, 1024, 64, 224),
                                     (7168, 1024, 128, 48), (2000, 2048, 256, 0), (500, 512, 200, 40)])
def test_linear_tcgen05_path(D, torch, M, K, N, h):
    """force_path = 3: tcgen05.mma (M=128 x N x K=16, TMEM accumulators) on SWIZZLE_128B SMEM operands
    (KC = 64), against the oracle."""
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(10, M + N), bias=True)
    y, sl, a = run_linear(D, torch, W, x, h, 64, bias=b, force_path=3)
    assert D.linear_query(a)["path"] == 3
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y), ref)


def test_linear_tcgen05_r_invariance_and_integer_exact(D, torch):
    """Integer inputs: exact sums -> bitwise equal to the oracle's RNE rounding; the output is the
    same bitwise for every split point (tier / CTA partition)."""
    M, K, N = 2000, 2048, 48
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(10, 5), kind="int")
    outs = []
    for h in (0, 64, 1000, 2000):
        y, _, _ = run_linear(D, torch, W, x, h, 64, force_path=3)
        outs.append(y)
    ref = Kx.split_linear(W[:0], W, x)
    assert np.array_equal(Kx.bf16_to_f64(outs[0]), Kx.round_to_bf16(ref))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("M,K,N,h", [(1024, 1024, 512, 64), (700, 2048, 384, 0), (300, 512, 257, 296),
                                     (7168, 1024, 512, 56)])
def test_linear_tcgen05_wide_n(D, torch, M, K, N, h):
    """N in (256, 512] (prefill-like batch): two N = 256 MMAs per K step into 512
    TMEM columns, x as two 256-row TMA boxes, one M tile per CTA -- vs the oracle; integer inputs
    bitwise, and bitwise independent of the tier split."""
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(12, M + N), bias=True)
    y, sl, a = run_linear(D, torch, W, x, h, 64, bias=b)
    q = D.linear_query(a)
    assert q["path"] == 3 and q["rows_per_cta_hbm_max"] <= 128
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(y), ref)
    Wi, xi, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(12, M), kind="int")
    outs = [run_linear(D, torch, Wi, xi, hh, 64)[0] for hh in (0, h, M - M % 8)]  # auto tcgen05: h % 8 == 0
    assert np.array_equal(Kx.bf16_to_f64(outs[0]), Kx.round_to_bf16(Kx.split_linear(Wi[:0], Wi, xi)))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("M,K,N,h", [(1024, 1024, 1024, 64), (700, 2048, 640, 0), (7168, 512, 1000, 256),
                                     (512, 512, 2048, 128), (300, 256, 4096, 0), (1000, 256, 3000, 504)])
def test_linear_tcgen05_pairs_w_multicast(D, torch, M, K, N, h):
    """N in (512, 4096]: groups of G = ceil(N / 512) CTAs share rows (rank r computes columns
    [512 r, 512 r + 512)). With cluster = 2 each group is a G-CTA cluster and rank 0 fetches every
    weight tile ONCE for all of it (bulk-copy multicast; a host tile crosses the link
    once); without it each CTA fetches its own copy (read amplification x G, Table 1). Outputs vs the oracle, bitwise equal with and
    without multicast, integer inputs bitwise exact."""
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(13, M + N), bias=True)
    ys = []
    for cl in (0, 2):
        y, sl, a = run_linear(D, torch, W, x, h, 64, bias=b, cluster=cl)
        q = D.linear_query(a)
        assert q["path"] == 3 and q["grid"] % (-(-N // 512)) == 0
        ys.append(y)
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
    from tests.gpu_util import assert_close
    assert_close(Kx.bf16_to_f64(ys[1]), ref)
    if h > 0:  # (h == 0 without a cluster takes the CTA-pair GEMM: checked against the oracle)
        assert np.array_equal(ys[0], ys[1])
    else:
        assert_close(Kx.bf16_to_f64(ys[0]), ref)
    Wi, xi, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(13, M), kind="int")
    yi = run_linear(D, torch, Wi, xi, h, 64, cluster=2)[0]
    assert np.array_equal(Kx.bf16_to_f64(yi), Kx.round_to_bf16(Kx.split_linear(Wi[:0], Wi, xi)))


@pytest.mark.parametrize("xf,N", [(1, 64), (1, 24), (2, 64), (2, 128)])
def test_linear_tcgen05_operand_transforms(D, torch, xf, N):
    """tcgen05 path with the fused pre-norm (RMSNorm) or SwiGLU operand applied in SMEM by the
    transform warps, against the oracle."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    M, K, h = 3584, 2048, 32
    W, _, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(11, M + N + xf))
    g = synth.rng(N * 7 + xf)
    sl = SplitLinear(D, W, h, 64)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    if xf == 1:
        x = synth.bf16_bits((g.standard_normal((N, K)) * 1.5 + 0.3).astype(np.float32))
        w_ln = synth.bf16_bits((1.0 + 0.2 * g.standard_normal(K)).astype(np.float32))
        xd, wd = to_dev(x), to_dev(w_ln)
        stats = torch.zeros((N, 4), dtype=torch.float32, device="cuda")
        D.row_stats(xd, N, K, stats)
        a = sl.args(xd, y, N, force_path=3)
        a.ln_w, a.ln_stats, a.ln_parts, a.ln_rms, a.ln_eps = wd.data_ptr(), stats.data_ptr(), 1, 1, 1e-5
        xf64 = Kx.bf16_to_f64(x)
        from oracle import layer as Ly  # noqa: F401
        hx = Kx.round_to_bf16(Kx.rmsnorm(xf64, Kx.bf16_to_f64(w_ln), 1e-5))
    else:
        x = synth.normal_bf16(g, (N, 2 * K), 1.5)
        xd = to_dev(x)
        a = sl.args(xd, y, N, force_path=3)
        a.x_swiglu = 1
        gf, uf = Kx.bf16_to_f64(x[:, :K]), Kx.bf16_to_f64(x[:, K:])
        hx = Kx.round_to_bf16(gf / (1.0 + np.exp(-gf)) * uf)
    assert D.linear_query(a)["path"] == 3
    D.linear(a)
    torch.cuda.synchronize()
    ref = Kx.split_linear(W[:h], W[h:], synth.bf16_bits(hx.astype(np.float32)))
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("fp", [3, 4])
@pytest.mark.parametrize("M,K,N,h", [(1280, 8192, 64, 0), (1024, 8192, 48, 32), (7168, 8192, 64, 48), (300, 2048, 16, 0),
                                     (8192, 1024, 64, 256), (8192, 3584, 64, 0), (7168, 1024, 128, 8)])
def test_linear_tcgen05_split_k(D, torch, M, K, N, h, fp):
    """tcgen05 with few rows per CTA: (row block, K split) items, fp32 partials in the caller's
    workspace, fixed-order combine kernel (bias / residual applied there), against the oracle.
    force_path 3: weight rows as the MMA's M (128-row blocks); 4: swapped operands (batch = M,
    128 or 256 weight rows = N per instruction, umma_swap_kernel)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(12, M + N), bias=True)
    g = synth.rng(M + N)
    res = synth.normal_bf16(g, (N, M), 1.0)
    sl = SplitLinear(D, W, h, 64)
    xd, bd, rd = to_dev(x), to_dev(b), to_dev(res)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    a = sl.args(xd, y, N, bias=bd, residual=rd, force_path=fp)
    ws = D.linear_workspace_size(a)
    assert ws > 0
    wsb = torch.zeros(ws, dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = wsb.data_ptr(), ws
    D.linear(a)
    torch.cuda.synchronize()
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b, residual_bits=res)
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("fp", [3, 4])
def test_linear_tcgen05_split_k_r_invariance_integer_exact(D, torch, fp):
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    M, K, N = 1280, 4096, 32
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(12, 3), kind="int")
    outs = []
    for h in (0, 128, 640):
        sl = SplitLinear(D, W, h, 64)
        xd = to_dev(x)
        y = torch.empty((N, M), dtype=torch.int16, device="cuda")
        a = sl.args(xd, y, N, force_path=fp)
        ws = D.linear_workspace_size(a)
        assert ws > 0
        wsb = torch.zeros(ws, dtype=torch.uint8, device="cuda")
        a.workspace, a.workspace_bytes = wsb.data_ptr(), ws
        D.linear(a)
        torch.cuda.synchronize()
        outs.append(from_dev(y))
    ref = Kx.split_linear(W[:0], W, x)
    assert np.array_equal(Kx.bf16_to_f64(outs[0]), Kx.round_to_bf16(ref))
    assert np.array_equal(outs[1], outs[0]) and np.array_equal(outs[2], outs[0])


def _run_cfg(D, torch, W, x, h, kc, **cfg):
    """Launch with a split-K workspace when the plan asks for one; returns (y bits, launch info)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    M, K = W.shape
    N = x.shape[0]
    sl = SplitLinear(D, W, h, kc)
    xd = to_dev(x)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    a = sl.args(xd, y, N, **cfg)
    wsb = None
    if kc == 64 and N > 16:
        a.workspace, a.workspace_bytes = 256, 1 << 40
        need = D.linear_workspace_size(a)
        a.workspace, a.workspace_bytes = None, 0
        if need:
            wsb = torch.zeros(need, dtype=torch.uint8, device="cuda")
            a.workspace, a.workspace_bytes = wsb.data_ptr(), need
    info = D.linear_query(a)
    D.linear(a)
    torch.cuda.synchronize()
    return from_dev(y), info


@pytest.mark.parametrize("M,K,N,h,kc", [(3000, 4096, 2, 400, 512), (3000, 4096, 8, 400, 256), (2048, 2048, 48, 512, 64),
                                        (7168, 8192, 64, 1024, 64)])
def test_linear_congestion_knobs_bitwise(D, torch, M, K, N, h, kc):
    """Congestion control is a performance mechanism only: the host window W, the
    host-CTA count, cc on / off, the HBM ring depth -- and, on split-K plans, the host-item gate --
    never change a bit of the output (FMA path at N = 2 is forced below; mma.sync at N = 8;
    tcgen05 at N = 48; tcgen05 split-K (swapped) at N = 64 with many host items)."""
    from tests.gpu_util import assert_close
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(30, M + N))
    fp = dict(force_path=1) if N <= 4 else {}
    base, info0 = _run_cfg(D, torch, W, x, h, kc, congestion_control=0, **fp)
    assert_close(Kx.bf16_to_f64(base), Kx.linear(W, x))
    gates = set()
    for knobs in (dict(congestion_control=1), dict(congestion_control=1, window=1), dict(congestion_control=1, window=3),
                  dict(congestion_control=1, n_cta_host=1), dict(congestion_control=1, n_cta_host=4),
                  dict(congestion_control=0, window=2, stages=3), dict(congestion_control=1, stages=2)):
        got, info = _run_cfg(D, torch, W, x, h, kc, **knobs, **fp)
        gates.add(info["host_gate"])
        assert np.array_equal(got, base), knobs
    if info0["ksplit"] > 1:  # the split-K host gate was active in some of the runs
        assert max(gates) >= 1


@pytest.mark.parametrize("M,K,N", [(28672, 7168, 32), (7168, 8192, 64)])
def test_linear_large_m_r_invariance_bitwise(D, torch, M, K, N):
    """tcgen05 at batch > 16: whether K is split is decided from (M, K, SM count) only, so the
    summation order of a row never depends on the tier split h (OPT fc1 shape: no split at any h;
    Llama TP8 o shape: split at every h) -- outputs bitwise equal for h in {0, 64, 1024, M/2}."""
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(31, M + N), kind="int")
    outs, splits = [], set()
    for h in (0, 64, 1024, M // 2):
        y, info = _run_cfg(D, torch, W, x, h, 64)
        outs.append(y)
        splits.add(info["ksplit"])
    assert len(splits) == 1
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert np.array_equal(Kx.bf16_to_f64(outs[0]), Kx.round_to_bf16(Kx.linear(W, x)))


@pytest.mark.parametrize("M,K,N,h", [(7168, 8192, 64, 1024), (1280, 4096, 32, 128)])
def test_linear_cta_rows_split_k_match_oracle(D, torch, M, K, N, h):
    """dak_linear_cta_rows on split-K plans: CTA j of a tier owns K split j % S of that tier's
    kblock-row block j // S (the oracle's rule, oracle/partition.py linear_splitk_items)."""
    from oracle import partition as Pt
    a = D.linear_args(16, 16, M, K, h, 64, N, 16, 16)
    a.workspace, a.workspace_bytes = 256, 1 << 40
    info = D.linear_query(a)
    assert info["ksplit"] > 1
    ref = Pt.linear_splitk_items(M, h, info["ksplit"], info["kblock"])
    got = [D.linear_cta_rows(a, c) for c in range(info["grid"])]
    assert got == ref


def test_linear_split_k_shared_workspace_reuse(D, torch):
    """One split-K workspace serves a chain of swapped-operand ops with different split counts,
    launched back to back without a host sync (each op's partials are written after its dependency
    wait and reduced before the next op runs): every output bit-exact (integer inputs) vs the oracle."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    shapes = [(1280, 8192, 64, 0), (8192, 1024, 64, 256), (7168, 4096, 64, 0), (1024, 2048, 48, 128)]
    runs = []
    for i, (M, K, N, h) in enumerate(shapes):
        W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(32, i), kind="int")
        sl = SplitLinear(D, W, h, 64)
        xd = to_dev(x)
        y = torch.empty((N, M), dtype=torch.int16, device="cuda")
        a = sl.args(xd, y, N, force_path=4)
        runs.append((W, x, sl, xd, y, a))
    need = max(D.linear_workspace_size(r[5]) for r in runs)
    wsb = torch.zeros(need, dtype=torch.uint8, device="cuda")
    for r in runs:
        r[5].workspace, r[5].workspace_bytes = wsb.data_ptr(), need
        assert D.linear_query(r[5])["ksplit"] > 1
    for _ in range(3):
        for r in runs:
            D.linear(r[5])
    torch.cuda.synchronize()
    for W, x, sl, xd, y, a in runs:
        assert np.array_equal(Kx.bf16_to_f64(from_dev(y)), Kx.round_to_bf16(Kx.linear(W, x)))


@pytest.mark.parametrize("N,kc,h", [(1, 512, 32), (1, 256, 0), (8, 256, 48), (16, 128, 64)])
def test_linear_chain_bitwise_vs_single_launches(D, torch, N, kc, h):
    """dak_linear_chain (persistent multi-op launch): a DEPENDENT chain of C1-shaped GEMVs (x of op i
    = y of op i-1, 4096 x 4096, host rows at the planner's share) and an independent tail of other
    shapes with bias / ReLU / residual give outputs bitwise equal to the ops launched one by one
    through dak_linear (mma.sync path, same kc and host CTAs); integer inputs are exact against the
    oracle. Run twice on one workspace (it must be left zeroed)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    M = K = 4096
    g = synth.rng(90 + N)
    Ws = [synth.linear_inputs(M, K, N, seed=synth.seed_for(40, i), kind="int")[0] for i in range(3)]
    x0 = synth.linear_inputs(M, K, N, seed=synth.seed_for(41, N), kind="int")[1]
    sls = [SplitLinear(D, W, h, kc) for W in Ws]
    bufs = [to_dev(x0)] + [torch.zeros((N, M), dtype=torch.int16, device="cuda") for _ in range(3)]
    # tail: independent ops of other shapes (same N, kc) with bias / ReLU / residual
    W2, x2, b2 = synth.linear_inputs(1024, 2048, N, seed=synth.seed_for(42, N), bias=True)
    res2 = synth.normal_bf16(g, (N, 1024), 1.0)
    sl2 = SplitLinear(D, W2, 16 if h else 0, kc)
    x2d, b2d, r2d = to_dev(x2), to_dev(b2), to_dev(res2)
    y2 = torch.zeros((N, 1024), dtype=torch.int16, device="cuda")
    cfg = dict(force_path=2, n_cta_host=2, congestion_control=1, pdl=1)
    ops = [sls[i].args(bufs[i], bufs[i + 1], N, **cfg) for i in range(3)]
    ops.append(sl2.args(x2d, y2, N, bias=b2d, residual=r2d, act=D.ACT_RELU, **cfg))
    ref = []
    for a, out in zip(ops, bufs[1:] + [y2]):
        D.linear(a)
        torch.cuda.synchronize()
        ref.append(from_dev(out).copy())
    for b in bufs[1:] + [y2]:
        b.zero_()
    ws = torch.zeros(64, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        D.linear_chain(ops, ws, ws.numel())
        torch.cuda.synchronize()
        for r_, out in zip(ref, bufs[1:] + [y2]):
            assert np.array_equal(from_dev(out), r_)
        assert int(ws.view(torch.int32).abs().sum()) == 0
    y1 = Kx.round_to_bf16(Kx.linear(Ws[0], x0))
    assert np.array_equal(Kx.bf16_to_f64(ref[0]), y1)


def _run_pair(D, torch, W, x, h, bias=None, residual=None, act=0, split=True, **cfg):
    """One CTA-pair GEMM launch (force_path 5), with the split-K workspace the plan asks for when
    `split`; returns (y bits, launch info)."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    M, K = W.shape
    N = x.shape[0]
    sl = SplitLinear(D, W, h, 64)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    # the device copies must outlive the launch (the args hold raw pointers)
    xd = to_dev(x)
    bd = to_dev(bias) if bias is not None else None
    rd = to_dev(residual) if residual is not None else None
    a = sl.args(xd, y, N, bias=bd, residual=rd, act=act, force_path=5, **cfg)
    wsb = None
    if split:
        a.workspace, a.workspace_bytes = 256, 1 << 40
        need = D.linear_workspace_size(a)
        a.workspace, a.workspace_bytes = None, 0
        if need:
            wsb = torch.zeros(need, dtype=torch.uint8, device="cuda")
            a.workspace, a.workspace_bytes = wsb.data_ptr(), need
    info = D.linear_query(a)
    D.linear(a)
    torch.cuda.synchronize()
    del xd, bd, rd, wsb
    return from_dev(y), info


@pytest.mark.parametrize("M,K,N,h,act,res", [(1024, 1024, 256, 0, 0, False), (700, 2048, 384, 0, 1, True),
                                             (7168, 512, 1000, 256, 0, False), (300, 256, 520, 40, 0, True),
                                             (2000, 2048, 130, 0, 0, False), (512, 512, 2048, 128, 1, False),
                                             (257, 4096, 512, 0, 0, False)])
def test_linear_cta_pair_gemm(D, torch, M, K, N, h, act, res):
    """The CTA-pair GEMM (force_path = 5; auto for h == 0 and N > 128): tcgen05.mma.cta_group::2 on
    256-row x 256/512-column pair tiles, both tiers, ragged M / N, with and without K splits (fp32
    partials + the reduce kernel), bias / ReLU / residual epilogue -- vs the oracle; integer inputs
    bitwise exact, and bitwise the same for every tier split h (the splits depend on M, N, K only)."""
    from tests.gpu_util import assert_close
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(41, M + N), bias=True)
    r = synth.normal_bf16(synth.rng(M + 3 * N), (N, M), 0.5) if res else None
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b, act="relu" if act else "none", residual_bits=r)
    splits = set()
    for split in (False, True):
        y, info = _run_pair(D, torch, W, x, h, bias=b, residual=r, act=act, split=split)
        assert info["path"] == 3 and info["grid"] % 2 == 0
        splits.add(info["ksplit"])
        assert_close(Kx.bf16_to_f64(y), ref)
    Wi, xi, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(41, M), kind="int")
    outs = [_run_pair(D, torch, Wi, xi, hh)[0] for hh in sorted({0, h, M // 2, M})]  # any h: no 8-row rule
    assert np.array_equal(Kx.bf16_to_f64(outs[0]), Kx.round_to_bf16(Kx.split_linear(Wi[:0], Wi, xi)))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_linear_cta_pair_chain_pdl_and_strided_y(D, torch):
    """Two CTA-pair GEMMs chained with programmatic dependent launch on one stream, the second
    reading the first's output as x (its x loads and y / residual accesses come after the dependency
    wait), the second writing into a wider row-strided y (ldy > M) with a residual -- vs the oracle."""
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    M1, K1, N = 1024, 768, 320       # y1 [N, M1] becomes x2 (K2 = M1)
    M2, K2 = 512, 1024
    g = synth.rng(4711)
    W1, x1, _ = synth.linear_inputs(M1, K1, N, seed=synth.seed_for(43, 1))
    W2, _, _ = synth.linear_inputs(M2, K2, N, seed=synth.seed_for(43, 2))
    ldy = M2 + 64
    res = synth.normal_bf16(g, (N, ldy), 0.5)
    sl1, sl2 = SplitLinear(D, W1, 0, 64), SplitLinear(D, W2, 0, 64)
    x1d = to_dev(x1)
    y1 = torch.empty((N, M1), dtype=torch.int16, device="cuda")
    y2 = to_dev(np.zeros((N, ldy), np.uint16))
    rd = to_dev(res)
    a1 = sl1.args(x1d, y1, N, pdl=1)
    a2 = D.linear_args(None, sl2.hbm, M2, K2, 0, 64, N, y1, y2, residual=rd, cfg=dict(pdl=1), ldy=ldy)
    wss = []
    for a in (a1, a2):
        a.workspace, a.workspace_bytes = 256, 1 << 40
        need = D.linear_workspace_size(a)
        a.workspace, a.workspace_bytes = None, 0
        if need:
            wss.append(torch.zeros(need, dtype=torch.uint8, device="cuda"))
            a.workspace, a.workspace_bytes = wss[-1].data_ptr(), need
        assert D.linear_query(a)["kblock"] == 256  # the CTA-pair plan
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            D.linear(a1, s)
            D.linear(a2, s)
    torch.cuda.synchronize()
    y1b = from_dev(y1)
    assert_close(Kx.bf16_to_f64(y1b), Kx.linear(W1, x1))
    ref2 = Kx.linear(W2, y1b) + Kx.bf16_to_f64(res)[:, :M2]
    got2 = from_dev(y2)
    assert_close(Kx.bf16_to_f64(got2[:, :M2]), ref2)
    assert np.array_equal(got2[:, M2:], np.zeros((N, ldy - M2), np.uint16))  # columns past M untouched
