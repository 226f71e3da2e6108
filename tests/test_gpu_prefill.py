"""GPU parity of dak_prefill_attention (causal prefill over the tier-split paged KV cache, SURVEY
§8(f) rank 3) against the float64 oracle (oracle/kernels.py paged_prefill_attention)."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2604_26074_b200 import dak
    return dak


def run_prefill(D, Ls, T, Hkv, Hq, page, frac, seed, kind="normal", cp=1, stage=True, **cfg):
    import torch
    from tests.gpu_util import make_paged_kv, PagedKV, to_dev, from_dev
    d = 128
    q, K, V, (kg, vg, kh, vh, bt), n_host = make_paged_kv(Ls, Hkv, d, page, frac, cp, seed, Hq * T, kind=kind)
    B = len(Ls)
    q = q.reshape(B, T, Hq, d)
    kv = PagedKV(D, kg, vg, kh, vh, bt, page)
    qd = to_dev(q)
    out = torch.full((B, T, Hq, d), 0x7FC0, dtype=torch.int16, device="cuda")  # NaN fill: every row must be written
    sl = torch.tensor(Ls, dtype=torch.int32, device="cuda")
    ws = None
    if stage:  # host streamer CTAs + device staging pool (each host page crosses the link once)
        ws = torch.empty(D.prefill_workspace_size(B, Hkv, page, bt.shape[1]), dtype=torch.uint8, device="cuda")
    D.prefill_attention(qd, out, kv.kg, kv.vg, kv.kh.dp, kv.vh.dp, kv.bt, sl, B, T, Hq, Hkv, d, page, bt.shape[1],
                        cfg=cfg, workspace=ws, workspace_bytes=ws.numel() if ws is not None else 0)
    torch.cuda.synchronize()
    ref = Kx.paged_prefill_attention(q, kg, vg, kh, vh, bt, Ls, page)
    return from_dev(out), ref, n_host


CASES = [  # (seq lens, T, Hkv, Hq, page, host fraction)
    ([200, 131], 131, 2, 16, 64, 0.5),     # GQA 8, one request is a full prompt (T = L)
    ([64, 300], 40, 4, 4, 64, 0.3),        # MHA, chunked prefill after a prefix
    ([1000], 77, 1, 8, 128, 0.5),          # Llama TP8 shard shape (1 kv head x 8 q heads), page 128
    ([129, 129, 129], 1, 2, 8, 64, 0.5),   # T = 1 is decode attention
    ([513], 200, 8, 64, 64, 1.0),          # all on the host, 64 q heads
    ([256], 256, 2, 4, 64, 0.0),           # all in HBM, rows a multiple of 128
]


@pytest.mark.parametrize("stage", [True, False])
@pytest.mark.parametrize("Ls,T,Hkv,Hq,page,frac", CASES)
def test_prefill_parity(D, Ls, T, Hkv, Hq, page, frac, stage):
    from tests.gpu_util import assert_close
    got, ref, _ = run_prefill(D, Ls, T, Hkv, Hq, page, frac, seed=700 + T, stage=stage)
    assert_close(Kx.bf16_to_f64(got), ref)


@pytest.mark.parametrize("Ls,T,Hkv,Hq,page,frac", CASES[:3] + CASES[4:5])
def test_prefill_mma_sync_form(D, Ls, T, Hkv, Hq, page, frac):
    """cfg.force_path = 2 selects the mma.sync (HMMA) form of the kernel: the same parity bar."""
    from tests.gpu_util import assert_close
    got, ref, _ = run_prefill(D, Ls, T, Hkv, Hq, page, frac, seed=800 + T, force_path=2)
    assert_close(Kx.bf16_to_f64(got), ref)


@pytest.mark.parametrize("kind", ["wide", "constk", "dominant"])
def test_prefill_score_ranges(D, kind):
    from tests.gpu_util import assert_close
    got, ref, _ = run_prefill(D, [333, 190], 100, 2, 16, 64, 0.5, seed=9, kind=kind)
    assert_close(Kx.bf16_to_f64(got), ref)


def test_prefill_r_invariance_and_stages_bitwise(D):
    """The same logical KV with 0 / 50 / 100 % of its pages on the host, any ring depth, host pages
    streamed through the staging pool or read directly, any streamer count: bitwise the same output
    (tiles are consumed newest keys first whatever their tier or path)."""
    base, _, _ = run_prefill(D, [700, 260], 120, 2, 16, 64, 0.0, seed=21)
    for frac, st, stage, nh in ((0.5, 0, True, 0), (1.0, 0, True, 1), (0.5, 2, False, 0), (0.0, 3, True, 0),
                                (1.0, 0, False, 0), (0.5, 0, True, 7)):
        got, _, _ = run_prefill(D, [700, 260], 120, 2, 16, 64, frac, seed=21, stages=st, stage=stage, n_cta_host=nh)
        assert np.array_equal(got, base), (frac, st, stage, nh)


def test_prefill_errors(D):
    import torch
    q = torch.zeros(16, dtype=torch.int16, device="cuda")
    with pytest.raises(D.DakError) as e:
        D.prefill_attention(q, q, q, q, None, None, q, q, 1, 1, 8, 2, 128, 32, 1)  # page 32
    assert e.value.code == "EUNSUPPORTED"
    with pytest.raises(D.DakError) as e:
        D.prefill_attention(q, q, q, q, None, None, q, q, 1, 1, 8, 3, 128, 64, 1)  # Hq % Hkv
    assert e.value.code == "EINVAL"
