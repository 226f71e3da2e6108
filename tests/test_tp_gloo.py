"""World-size-2 CPU test of the tensor-parallel path's host logic (gloo): every rank shards the
Llama layer with paper_2604_26074_b200.tp.shard_llama, computes its partial o / down outputs with
the oracle on its shard, the partials are all-reduced with torch.distributed (the exchange
dak_allreduce_residual performs over NCCL on GPUs), and the result equals the unsharded oracle."""
import os
import socket

import numpy as np
import pytest

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from oracle import layer as Ly
    from paper_2604_26074_b200 import tp
    from tests.test_oracle_llama import make_llama_params
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.rng(77)
        H, F, nh, nkv, d, B = 256, 512, 4, 2, 64, 3
        p = make_llama_params(g, 1, H, F, 60, nh, nkv, d)
        x = g.standard_normal((B, H))
        Kp = [synth.normal_bf16(g, (4 + b, nkv, d)) for b in range(B)]
        Vp = [synth.normal_bf16(g, (4 + b, nkv, d)) for b in range(B)]
        pos = np.array([4, 5, 6])
        full = {k.split(".", 1)[1]: v for k, v in p.items() if k.startswith("L0.")}
        ref, _, _ = Ly.llama_decode_layer(x, full, Kp, Vp, pos, nh, nkv)
        loc = tp.shard_llama(p, rank, world, nh, nkv, d)
        lp = {k.split(".", 1)[1]: v for k, v in loc.items() if k.startswith("L0.")}
        kv = tp.shard_range(nkv, rank, world)
        Kl = [k[:, kv] for k in Kp]
        Vl = [v[:, kv] for v in Vp]
        dims = tp.local_dims(nh, nkv, F, 60, world)
        (attn_part, mlp_fn), _, _ = Ly.llama_decode_layer(x, lp, Kl, Vl, pos, dims["n_heads"], dims["n_kv"], shard=(0, 1))
        t = torch.from_numpy(attn_part.copy())
        dist.all_reduce(t)
        x1 = x + t.numpy()
        t = torch.from_numpy(mlp_fn(x1).copy())
        dist.all_reduce(t)
        x2 = x1 + t.numpy()
        q.put((rank, float(np.abs(x2 - ref).max()), float(np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


def test_tp_world2_gloo_matches_unsharded():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, err, scale in res:
        assert err <= 1e-10 * max(1.0, scale), (rank, err)


def test_shard_ranges_cover_weights():
    from paper_2604_26074_b200 import tp
    g = synth.rng(3)
    from tests.test_oracle_llama import make_llama_params
    p = make_llama_params(g, 1, 64, 128, 16, 4, 2, 16)
    parts = [tp.shard_llama(p, r, 2, 4, 2, 16) for r in range(2)]
    for name in ("L0.q", "L0.k", "L0.v", "L0.gate", "L0.up", "lm_head"):
        assert np.array_equal(np.concatenate([pt[name] for pt in parts], axis=0), p[name])
    for name in ("L0.o", "L0.down"):
        assert np.array_equal(np.concatenate([pt[name] for pt in parts], axis=1), p[name])
    with pytest.raises(ValueError):
        tp.shard_range(6, 0, 4)
