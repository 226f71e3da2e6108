"""GPU tests of the host tier and the attention auto configuration: NUMA-bound pinned pages
(dak_host_alloc with a node) are read by the split kernels exactly like
cudaHostAlloc pages; dak_attention with n_cta_host = 0 picks its host CTAs from the block table
and gives bitwise the same result as any explicit count."""
import ctypes
import os

import numpy as np
import pytest

import synth
from oracle import kernels as Kx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2604_26074_b200 import dak
    return dak


def _page_node(addr: int) -> int:
    """get_mempolicy(MPOL_F_NODE | MPOL_F_ADDR): the node backing the page at addr."""
    libc = ctypes.CDLL(None, use_errno=True)
    node = ctypes.c_int(-1)
    SYS_get_mempolicy = 239  # x86_64
    r = libc.syscall(SYS_get_mempolicy, ctypes.byref(node), None, ctypes.c_ulong(0), ctypes.c_void_p(addr),
                     ctypes.c_ulong(3))
    return node.value if r == 0 else -2


def test_numa_bound_host_alloc(D):
    import torch
    node = D.device_numa_node()
    use = max(node, 0)
    hp, dp = D.host_alloc(8 << 20, numa_node=use)
    assert hp and dp
    if os.uname().machine == "x86_64":
        got = _page_node(hp)
        assert got in (use, -2), got
    # the kernels read NUMA-bound pages like any mapped host memory: a split GEMV over them
    from tests.gpu_util import to_dev, from_dev, assert_close
    M, K, N, h = 512, 2048, 4, 128
    W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(40, 1))
    Wd = to_dev(W)
    D.pack_linear(Wd[:h].contiguous(), h, K, 256, dp)
    hbm = torch.empty((M - h) * K, dtype=torch.int16, device="cuda")
    D.pack_linear(Wd[h:].contiguous(), M - h, K, 256, hbm)
    y = torch.empty((N, M), dtype=torch.int16, device="cuda")
    xd = to_dev(x)
    D.linear(D.linear_args(dp, hbm, M, K, h, 256, N, xd, y))
    torch.cuda.synchronize()
    assert_close(Kx.bf16_to_f64(from_dev(y)), Kx.linear(W, x))
    D.host_free(hp)
    with pytest.raises(D.DakError):
        D.host_alloc(4096, write_combined=True, numa_node=use)


@pytest.mark.parametrize("Ls,frac,cp", [([900, 40, 2000], 0.5, 2), ([300, 301], 0.0, 1), ([513], 1.0, 2)])
def test_attention_auto_host_ctas_bitwise(D, Ls, frac, cp):
    """n_cta_host = 0: the kernel counts the host units in the block table and sizes the host CTAs
    (one per 4 units, <= 16, none without host units); output bitwise equal to explicit counts and
    within tolerance of the oracle."""
    import torch
    from tests.gpu_util import assert_close
    from tests.test_gpu_attention import run_attn
    auto, ref, _ = run_attn(D, torch, Ls, 2, 8, 64, cp, frac, seed=71, n_cta_host=0)
    assert_close(Kx.bf16_to_f64(auto), ref)
    for nh in (1, 3):
        got, _, _ = run_attn(D, torch, Ls, 2, 8, 64, cp, frac, seed=71, n_cta_host=nh)
        assert np.array_equal(got, auto)


def test_calibrate_sweep_and_choice(D):
    """dak_calibrate (the parameter-sweeping profiler run before the kernels): on the
    B200's PCIe link the probe measures an HBM rate near the copy peak with every SM on HBM, a link
    rate of tens of GB/s that rises with the bytes in flight, a positive link latency, and its choice
    is dak_calib_select's over the table it returns."""
    import torch
    hbm = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    hp, dp = D.host_alloc(64 << 20)
    try:
        n_host, window = (1, 2, 4), (1, 2, 4, 8)
        res, tab = D.calibrate(hbm, hbm.numel(), dp, 64 << 20, n_host=n_host, window=window, duration_us=200, reps=3)
    finally:
        D.host_free(hp)
    assert 3e12 < res["hbm_alone_bps"] < 9e12
    assert 1e10 < res["link_bps"] < 1e11 and 3e12 < res["hbm_bps"] < 9e12
    assert 0 < res["host_latency_s"] < 50e-6
    i, j = D.calib_select(tab, n_host, window, 0.005)
    assert (res["n_cta_host"], res["window"]) == (n_host[i], window[j])
    assert res["host_inflight_bytes"] == n_host[i] * window[j] * 16384
    assert tab[0, -1].sum() > tab[0, 0].sum()  # one host CTA: more requests in flight, a faster op
