"""Tensor-parallel combine over NCCL through the C ABI (BASELINE north_star: TP over 8 x B200).

- dak_allgather_cols on one GPU (NULL communicator and a 1-rank NCCL communicator);
- with >= 2 GPUs: `world` processes (one per GPU) each run their Megatron shard of a Llama decode
  step (DakLlama, dak_layer with a real multi-rank communicator: the row-parallel o / down partials
  are all-reduced by dak_allreduce_residual over NVLink), and every rank's vocabulary shard of the
  logits is compared with the unsharded oracle (oracle/layer.py llama_decode_step); the ranks'
  column-parallel GEMV shards are all-gathered with dak_allgather_cols and compared with the full
  oracle GEMV. Skipped on a one-GPU box (the driver's GPU tier has one GPU).
"""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly

pytestmark = pytest.mark.gpu


def _n_gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("N,Ml,use_comm", [(1, 4096, False), (5, 1024, False), (1, 4096, True), (5, 1024, True)])
def test_allgather_cols_one_rank(N, Ml, use_comm):
    import torch
    from paper_2604_26074_b200 import dak
    comm = dak.comm_init(dak.comm_unique_id(), 0, 1) if use_comm else None
    assert dak.comm_size(comm) == 1
    src = torch.randn(N, Ml, device="cuda").to(torch.bfloat16)
    dst = torch.empty_like(src)
    scratch = torch.empty_like(src)
    dak.allgather_cols(comm, src, dst, scratch, N, Ml)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    if comm:
        dak.comm_destroy(comm)


def test_nvls_needs_a_multicast_team():
    """dak_nvls_create refuses a one-rank communicator cleanly (EUNSUPPORTED: the engine keeps the
    ncclAllReduce combine), and the combine kernel rejects bad shapes."""
    from paper_2604_26074_b200 import dak
    comm = dak.comm_init(dak.comm_unique_id(), 0, 1)
    with pytest.raises(dak.DakError) as e:
        dak.nvls_create(comm, 1 << 20, 64)
    assert e.value.code in ("EUNSUPPORTED",)
    dak.comm_destroy(comm)
    with pytest.raises(dak.DakError):
        dak.nvls_residual_rmsnorm(None, 0, None, 4, 8192, None, 1e-5, None)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_worker(rank, world, uid, q):
    import torch
    from paper_2604_26074_b200 import dak, tp
    from paper_2604_26074_b200.engine import HW
    from paper_2604_26074_b200.llama import DakLlama, LlamaConfig
    from tests.gpu_util import SplitLinear, to_dev, from_dev
    from tests.test_oracle_llama import make_llama_params
    torch.cuda.set_device(rank)
    try:
        comm = dak.comm_init(uid, rank, world)
        assert dak.comm_size(comm) == world
        L, H, F, V, nh, nkv, d, B, ctx = 2, 1024, 2048, 256, 8, 8, 128, 4, 90
        g = synth.rng(5151)
        p = make_llama_params(g, L, H, F, V, nh, nkv, d)
        Kc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
        Vc = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(B)] for _ in range(L)]
        tokens = (np.arange(B) * 13 + 3) % V
        ref, _ = Ly.llama_decode_step(tokens, np.full(B, ctx - 1), p, Kc, Vc, nh, nkv)
        dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16)).cuda().view(torch.bfloat16)
               for k, v in p.items()}
        cfg = LlamaConfig(n_layers=L, hidden=H, n_heads=nh, n_kv_heads=nkv, ffn=F, vocab=V, name="llama-tp")
        hw = HW(hbm_bps=6555.5e9, link_bps=51.5e9)
        eng = DakLlama(cfg, B, ctx, hw, tp_rank=rank, tp_size=world, comm=comm, mode=dak.PLAN_EXACT,
                       y_req=int(0.05 * 2 * L * (4 * H * H + 3 * F * H) / world), page_size=64, chunk_pages=1,
                       weights=dev)
        kvr = tp.shard_range(nkv, rank, world)
        eng.load_kv([[k[:, kvr] for k in layer] for layer in Kc], [[v[:, kvr] for v in layer] for layer in Vc])
        eng.tokens.copy_(torch.from_numpy(tokens.astype(np.int32)))
        s = torch.cuda.Stream()
        eng.capture(s)
        eng.graph.replay()
        torch.cuda.synchronize()
        got = Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16))
        vr = tp.shard_range(V, rank, world)
        ref_shard = ref[:, vr]
        eng.close()
        # column-parallel GEMV (C5 TP form): rank r computes rows [r M/n, (r+1) M/n), 10% host
        M, K, N = 4096, 2048, 3
        W, x, _ = synth.linear_inputs(M, K, N, seed=synth.seed_for(5, 0))
        Ml = M // world
        Wl = W[rank * Ml:(rank + 1) * Ml]
        sl = SplitLinear(dak, Wl, 32, 256)
        yl = torch.empty((N, Ml), dtype=torch.int16, device="cuda")
        xd = to_dev(x)
        dak.linear(sl.args(xd, yl, N))
        y = torch.empty((N, M), dtype=torch.int16, device="cuda")
        scratch = torch.empty((world, N, Ml), dtype=torch.int16, device="cuda")
        dak.allgather_cols(comm, yl, y, scratch, N, Ml)
        torch.cuda.synchronize()
        yg = Kx.bf16_to_f64(from_dev(y))
        # NVLS combine (unfused TP path, batch 24): the same layer with the switch reduction
        nv_res = None
        Bn = 24
        tok_n = (np.arange(Bn) * 7 + 1) % V
        Kn = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(Bn)] for _ in range(L)]
        Vn = [[synth.normal_bf16(g, (ctx - 1, nkv, d)) for _ in range(Bn)] for _ in range(L)]
        try:
            eng2 = DakLlama(cfg, Bn, ctx, hw, tp_rank=rank, tp_size=world, comm=comm, mode=dak.PLAN_EXACT, y_req=0,
                            page_size=64, chunk_pages=1, weights=dev, nvls=True)
        except dak.DakError as e:
            nv_res = ("unsupported", str(e))
        else:
            eng2.load_kv([[k[:, kvr] for k in layer] for layer in Kn], [[v[:, kvr] for v in layer] for layer in Vn])
            eng2.tokens.copy_(torch.from_numpy(tok_n.astype(np.int32)))
            eng2.capture(s)
            eng2.graph.replay()
            torch.cuda.synchronize()
            got2 = Kx.bf16_to_f64(eng2.logits.view(torch.int16).cpu().numpy().view(np.uint16))
            ref2, _ = Ly.llama_decode_step(tok_n, np.full(Bn, ctx - 1), p, Kn, Vn, nh, nkv)
            nv_res = (got2, ref2[:, vr])
            eng2.close()
        q.put((rank, got, ref_shard, yg, Kx.linear(W, x), nv_res))
        dak.comm_destroy(comm)
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, "error", traceback.format_exc(), None, None, None))


@pytest.mark.parametrize("world", [2, 8])
def test_tp_layer_multi_rank_matches_oracle(world):
    if _n_gpus() < world:
        pytest.skip(f"needs {world} GPUs (this box has {_n_gpus()})")
    import torch.multiprocessing as mp
    from paper_2604_26074_b200 import dak
    from tests.gpu_util import assert_close
    uid = dak.comm_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, uid, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=120)
    for rank, got, ref, yg, yref, nv in res:
        assert not isinstance(got, str), ref
        assert_close(got, ref, rtol=3e-2)
        assert_close(yg, yref)
        if nv[0] != "unsupported":  # NVSwitch box: the NVLS combine must match the oracle too
            assert_close(nv[0], nv[1], rtol=3e-2)
