"""GPU edge cases of the split operators against the oracle: tiny and ragged shapes, all-host and
all-HBM splits, single-token / single-page attention, each compute path (FMA, mma.sync, tcgen05,
tcgen05 split-K), and the ABI's error returns on bad launches."""
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


def _lin(D, torch, M, K, N, h, kc, **cfg):
    from tests.gpu_util import SplitLinear, to_dev, from_dev, assert_close
    W, x, b = synth.linear_inputs(M, K, N, seed=synth.seed_for(20, M * 31 + K + N + h), bias=True)
    sl = SplitLinear(D, W, h, kc)
    xd, bd = to_dev(x), to_dev(b)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    a = sl.args(xd, y, N, bias=bd, **cfg)
    wsb = None
    ws = D.linear_workspace_size(a) if cfg.get("force_path") == 3 else 0
    if ws:
        wsb = torch.zeros(ws, dtype=torch.uint8, device="cuda")
        a.workspace, a.workspace_bytes = wsb.data_ptr(), ws
    D.linear(a)
    torch.cuda.synchronize()
    ref = Kx.split_linear(W[:h], W[h:], x, bias_bits=b)
    assert_close(Kx.bf16_to_f64(from_dev(y)), ref)


@pytest.mark.parametrize("M,K,N,h,kc,path", [
    (1, 64, 1, 0, 64, 2), (1, 64, 1, 1, 64, 2), (7, 128, 3, 7, 64, 2), (16, 64, 16, 8, 64, 2),
    (100, 192, 4, 50, 64, 1), (3, 4096, 2, 1, 1024, 1), (149, 512, 8, 0, 128, 0),
    (8, 128, 24, 0, 64, 3), (24, 64, 64, 8, 64, 3), (136, 1024, 17, 128, 64, 3), (2000, 64, 33, 16, 64, 3)])
def test_linear_tiny_and_ragged(D, torch, M, K, N, h, kc, path):
    _lin(D, torch, M, K, N, h, kc, force_path=path)


@pytest.mark.parametrize("Ls,frac,cp", [([1], 0.0, 1), ([1, 2, 3], 1.0, 1), ([64], 1.0, 1), ([65, 1], 0.5, 1),
                                        ([700], 0.5, 4), ([16, 4000], 0.25, 16)])
def test_attention_edges(D, torch, Ls, frac, cp):
    from tests.gpu_util import assert_close
    from tests.test_gpu_attention import run_attn
    got, ref, _ = run_attn(D, torch, Ls, 2, 16, 64, cp, frac, seed=sum(Ls) + cp)
    assert_close(Kx.bf16_to_f64(got), ref)


@pytest.mark.parametrize("kind", ["wide", "constk", "dominant"])
@pytest.mark.parametrize("Ls,frac,cp", [([1, 90, 700], 0.5, 2), ([4000, 33], 0.25, 4)])
def test_attention_score_ranges(D, torch, kind, Ls, frac, cp):
    """Large / peaked / flat score distributions (synth.kv_inputs kinds): scores spanning +-100
    exercise the online-softmax rescaling inside a unit and the combine's running max across
    split-KV chunks; constant K makes every weight equal (o = mean V); one dominant key makes
    o ~ V of that token. Same per-element tolerance as every parity test."""
    from tests.gpu_util import assert_close
    from tests.test_gpu_attention import run_attn
    got, ref, _ = run_attn(D, torch, Ls, 2, 16, 64, cp, frac, seed=5 + sum(Ls), kind=kind)
    assert_close(Kx.bf16_to_f64(got), ref)


def test_linear_errors(D, torch):
    from tests.gpu_util import SplitLinear, to_dev
    W, x, _ = synth.linear_inputs(64, 128, 2, seed=1)
    sl = SplitLinear(D, W, 0, 64)
    xd = to_dev(x)
    y = torch.empty((2, 64), dtype=torch.int16, device="cuda")
    bad = sl.args(xd, y, 2, force_path=1)
    bad.N = 5  # CUDA-core path supports N <= 4
    with pytest.raises(D.DakError):
        D.linear(bad)
    a = sl.args(xd, y, 2, force_path=3)
    a.kc = 128  # tcgen05 needs kc == 64
    with pytest.raises(D.DakError):
        D.linear(a)
    a = sl.args(xd, y, 2)
    a.ldy = 10  # ldy < M
    with pytest.raises(D.DakError):
        D.linear(a)
