"""DAK decode hot-path benchmark (driver contract; see DESIGN.md §7 "Measurement").

Default workload (BASELINE.json configs[1]): OPT-30B decode step, batch 8, context 64 (prompt 32 +
32 decoded), weights split HBM / pinned host memory at the planner's BALANCED ratios
(every memory-bound op at its turning point B_l/(B_g+B_l)), one CUDA graph per step
(P:L637). A step = embed -> 48 x (QKV split-GEMM with the fused pre-norm, split attention with the
fused KV append, O split-GEMM + residual, FC1 split-GEMM (fused pre-norm) + ReLU, FC2 split-GEMM +
residual) -> LN -> LM head.

metric: aggregate GB/s = (weight + KV bytes read from HBM and host per step) / step time.
Also reported: decode tokens/s, per-tier bytes, roofline of the dominant kernel (dak_linear),
the CPU oracle baseline, clocks, and an end-to-end number with host buffers.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload llama3-70b-tp8]
Under torchrun every rank runs an independent replica (weak scaling, no data-path collective).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aggregate GB/s (HBM+host link) vs roofline; decode tokens/s at 1/2/4/8 B200"
LINK_GBS_DEFAULT = 51.5  # profiles/r01/calib_loadpath.jsonl: SM bulk-copy read of pinned host memory


def planner_rates(hbm_gbs, link_gbs):
    """Rates the planner balances (reading R10): what the split kernel itself sustains on this box
    -- HBM read stream with no host share and the host link at the balanced ratio -- from the
    committed C5 sweep (tools/sweep.py c5 -> profiles/r*/sweep_c5_ratio.jsonl); else the peaks."""
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "sweep_c5_ratio.jsonl")))
    if not files:
        return hbm_gbs, link_gbs, "peaks"
    pts = [json.loads(l) for l in open(files[-1]) if l.strip()]
    fc1 = [d for d in pts if d.get("M") == 28672 and d.get("cc") == 1]
    h0 = [d["gbs"] for d in fc1 if d["r"] == 0.0]
    rs = link_gbs / (hbm_gbs + link_gbs)
    near = sorted((d for d in fc1 if d["r"] > 0), key=lambda d: abs(d["r"] - rs))
    if not h0 or not near:
        return hbm_gbs, link_gbs, "peaks"
    return h0[0], near[0]["host_gbs"], os.path.relpath(files[-1], ROOT)


def measured_peaks():
    hbm, link = None, None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    try:
        best = 0.0
        with open(os.path.join(ROOT, "profiles", "r01", "calib_loadpath.jsonl")) as f:
            for line in f:
                r = json.loads(line)
                if r.get("test") in ("host_bulk", "host_tma"):
                    best = max(best, r.get("host_gbs", 0.0))
        link = best or None
    except Exception:
        pass
    return (hbm or 6650.0), (link or LINK_GBS_DEFAULT), ("measured" if hbm else "fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int, path: str):
        self.path = path
        self.p = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["unavailable"])
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=mx, reasons=sorted(reasons),
                    samples=len(sm))


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def reduce_max(v: float, world: int) -> float:
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------------------------
# CPU oracle baseline (the oracle as it stands; a bounded sample of the same workload)
# ------------------------------------------------------------------------------------------------
_CACHE = {}
READ_PEAK_GBS = 7381.6  # bulk-copy read ring, calibrated on the pool's B200 (profiles/r01/calib_loadpath.jsonl)


def oracle_sample(batch: int, min_seconds: float = 10.0):
    """OPT-30B layer-0 operators (q/k/v/o, fc1, fc2 as float64 oracle linears at N=batch, plus the
    layer's decode attention for all 56 heads over the 64-token context), repeated until
    >= min_seconds of CPU work. Returns (GB/s of algorithmic bytes, seconds, bytes, threads)."""
    import numpy as np
    import synth
    from oracle import kernels as Kx
    key = ("oracle_inputs", batch)
    if key not in _CACHE:  # seeded inputs drawn once per process (drawing 1.2 GB is not the oracle)
        g = np.random.default_rng(synth.seed_for(1, 0))
        H, F, heads, ctx = 7168, 28672, 56, 64
        shapes = [(3 * H, H), (H, H), (F, H), (H, F)]
        mats = [synth.normal_bf16(g, s, 1.0 / np.sqrt(s[1])) for s in shapes]
        xs = [synth.normal_bf16(g, (batch, s[1])) for s in shapes]
        q, K, V = synth.kv_inputs([ctx] * batch, heads, 128, heads, seed=synth.seed_for(1, 1))
        _CACHE[key] = (mats, xs, q, K, V)
    mats, xs, q, K, V = _CACHE[key]
    nbytes = sum(m.size * 2 for m in mats) + sum(k.size * 2 * 2 for k in K)
    t0 = time.perf_counter()
    reps = 0
    while True:
        for W, x in zip(mats, xs):
            Kx.linear(W, x)
        Kx.attention_dense(q, K, V)
        reps += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
    return nbytes * reps / dt / 1e9, dt, nbytes * reps, threads, reps


def in_step_profile(eng, stream, torch, dak, reps: int = 5) -> dict:
    """Per-kind time inside one decode step (see the roofline block in main)."""
    import numpy as np
    n_launch = eng.kernels_per_step() + 16
    buf = torch.zeros(n_launch * 1024 * 4, dtype=torch.int64, device="cuda")
    dak.trace_enable(buf, n_launch)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream), torch.cuda.graph(g, stream=stream):
            eng.enqueue_step(stream)
        meta = dak.trace_launches()
    finally:
        dak.trace_enable(None, 0)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    by_kind, steps = {}, []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        buf.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        steps.append(e0.elapsed_time(e1) / 1e3)
        T = buf.view(-1, 1024, 4).cpu().numpy()
        prev_end = None
        for i, m in enumerate(meta):
            st = T[i, :min(m["grid"], 1024)]
            ok = st[:, 3] > 0
            if not ok.any():
                continue
            end = float(st[ok, 3].max())
            if prev_end is None:  # the first launch: from its first CTA's start
                prev_end = float(st[st[:, 0] > 0, 0].min())
            by_kind[m["kind"]] = by_kind.get(m["kind"], 0.0) + max(0.0, end - prev_end) * 1e-9
            prev_end = max(prev_end, end)
    by_kind = {k: v / reps for k, v in by_kind.items()}
    return dict(linear_s=by_kind.get("linear", 0.0), by_kind_s=by_kind, traced_step_s=float(np.median(steps)),
                launches=len(meta))


def run_reference(a):
    """--impl reference: the CPU oracle on bounded samples of the same workload (rank 0 only)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(a.warmup):
        oracle_sample(a.batch, min_seconds=0.0)
    gbs = []
    t_all = 0.0
    for _ in range(a.steps):
        v, dt, nb, threads, reps = oracle_sample(a.batch, min_seconds=0.0)
        gbs.append(v)
        t_all += dt
    value = statistics.median(gbs)
    ms = t_all / a.steps * 1e3
    sample = "OPT-30B layer 0: q/k/v/o, fc1, fc2 float64 oracle linears at N=%d + decode attention (56 heads, 64 tokens)" % a.batch
    line = dict(metric=METRIC, value=round(value, 3), unit="GB/s", n_gpus=world, steps=a.steps, warmup=a.warmup,
                ms_per_step=round(ms, 3), higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic", impl="reference",
                config=dict(workload="opt-30b-decode-b%d-ctx%d" % (a.batch, a.context), model_shape="OPT-30B",
                            batch=a.batch, context=a.context, layers=48,
                            execution="CPU oracle (float64) on a bounded sample of the step: " + sample),
                cpu_baseline=dict(value=round(value, 3), unit="GB/s", cores=threads, kind="oracle", sample=sample),
                e2e=dict(value=round(value, 3), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                gpu_launches=0)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
def make_llama(a, hw, world, rank, dak, cal_kw=None):
    """BASELINE configs[2]: Llama-3-70B decode, batch 64, 64k context, TP8. Weights + KV of one rank
    (17.6 GB + 171.8 GB) exceed HBM, so the global ratio is forced by capacity (EXACT mode)
    against an HBM budget of 168 GB (12 GB kept for workspace); the default run is an 8-layer subset
    with the budget scaled by 8/80 (labelled; per-step time extrapolates x10). On one GPU the rank
    is rank 0 of 8 and its row-parallel all-reduce runs on a 1-rank NCCL communicator."""
    from paper_2604_26074_b200.llama import DakLlama, LLAMA3_70B
    from dataclasses import replace
    layers = a.layers or 8
    cfg = replace(LLAMA3_70B, n_layers=layers)
    tp_size = 8 if world == 1 else world
    batch = a.batch if a.batch != 8 else 64
    context = a.context if a.context != 64 else 65536
    saved = os.dup(1)  # NCCL may print its version banner on stdout: keep stdout one JSON line
    os.dup2(2, 1)
    try:
        if world == 1:
            comm = dak.comm_init(dak.comm_unique_id(), 0, 1)
        else:
            import torch.distributed as dist
            uid = [dak.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = dak.comm_init(uid[0], rank, world)
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    # a1: footprint of this rank's shard -> host bytes the HBM budget forces out, from the
    # library's own op profile (dak_decode_ops C_i: linear weights + KV) and dak_global_offload_bytes
    m = dak.model(dak.MODEL_LLAMA, layers, cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn, cfg.vocab,
                  tp_size=tp_size)
    ops = dak.decode_ops(m, batch, context, 16, 1024, hw.peak_flops, hw.peak_flops)
    w_bytes = sum(o["total_bytes"] for o in ops if o["role"] != "attn")
    kv_bytes = sum(o["total_bytes"] for o in ops if o["role"] == "attn")
    budget = int(168e9 * layers / cfg.__class__().n_layers)
    y_req, R = dak.global_offload_bytes(w_bytes, kv_bytes, budget)
    eng = DakLlama(cfg, batch, context, hw, tp_rank=rank, tp_size=tp_size, comm=comm, mode=dak.PLAN_EXACT,
                   y_req=y_req, pdl=not a.no_pdl, congestion_control=not a.no_cc, seed=1234 + rank,
                   chunk_pages=a.chunk_pages, nvls=a.nvls and world > 1, **(cal_kw or {}))
    wl = dict(workload="llama3-70b-tp8-b%d-ctx%d" % (batch, context), model_shape="Llama-3-70B (TP%d shard)" % tp_size,
              batch=batch, context=context, layers=layers, layers_model=80,
              extrapolation="x%d per token step" % (80 // layers) if layers != 80 else None,
              hbm_budget_bytes=budget, y_req_bytes=y_req, plan="EXACT (capacity-forced R=%.4f)" % R,
              tp="rank 0 of %d on one GPU (1-rank NCCL all-reduce)" % tp_size if world == 1 else "TP%d over NCCL" % world)
    eng.comm_handle = comm
    return eng, cfg, wl


def spawn_ranks(n: int):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks (one process per GPU)
    under torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dak", choices=["dak", "reference"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--context", type=int, default=64)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-cc", action="store_true")
    ap.add_argument("--chunk-pages", type=int, default=0, help="split-KV chunk in pages (0: the engine's rule)")
    ap.add_argument("--nvls", action="store_true", help="Llama TP (>= 2 ranks): NVLS combine instead of ncclAllReduce")
    ap.add_argument("--ratio", type=float, default=None, help="force global offload ratio R (EXACT mode)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--calibrate", action="store_true",
                    help="run dak_calibrate (P:L533-535) first: planner rates and congestion control from the sweep")
    ap.add_argument("--l2-prefetch-mb", type=float, default=0.0, help="L2 warm-up of the next linear (0: off)")
    ap.add_argument("--no-evict-first", action="store_true")
    ap.add_argument("--no-fuse-norm", action="store_true", help="LayerNorm kernels instead of the fused pre-norm")
    ap.add_argument("--plan-link-gbs", type=float, default=None,
                    help="host-link rate the planner assumes (default: the calibrated peak)")
    ap.add_argument("--plan-hbm-gbs", type=float, default=None, help="HBM rate the planner assumes")
    ap.add_argument("--plan-host-latency-us", type=float, default=0.0,
                    help="host-path latency the planner charges an op reading host bytes (latency-aware mode)")
    ap.add_argument("--layers", type=int, default=None,
                    help="layers (default: all 48 for OPT-30B; 8 of 80 for the Llama subset, labelled)")
    ap.add_argument("--workload", default="opt30b", choices=["opt30b", "llama3-70b-tp8"],
                    help="opt30b: BASELINE configs[1] (the bench line); llama3-70b-tp8: configs[2], this GPU's TP "
                         "shard (rank 0 of 8 on one GPU, or the real ranks under torchrun), capacity-forced ratios")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(a.gpus)
    if a.impl == "reference":
        return run_reference(a)

    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, HW, OPT_30B, OPTConfig

    world, rank, local = dist_setup()
    hbm_gbs, link_gbs, peak_src = measured_peaks()
    ph, pl, plan_src = planner_rates(hbm_gbs, link_gbs)
    hw = HW(hbm_bps=(a.plan_hbm_gbs or ph) * 1e9, link_bps=(a.plan_link_gbs or pl) * 1e9,
            host_latency_s=a.plan_host_latency_us * 1e-6)
    cal = None
    if a.calibrate:  # the online calibration sweep, before any decode kernel
        hbm_buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        hp, dp = dak.host_alloc(256 << 20, numa_node=dak.device_numa_node())
        try:
            cal, _ = dak.calibrate(hbm_buf, hbm_buf.numel(), dp, 256 << 20)
        finally:
            dak.host_free(hp)
        del hbm_buf
        torch.cuda.empty_cache()
        hw = HW.from_calibration(cal)
        plan_src = "dak_calibrate"
    cal_kw = dict(n_cta_host=max(1, cal["n_cta_host"]), host_inflight_kb=int(cal["host_inflight_bytes"] // 1024)) if cal else {}
    llama = a.workload == "llama3-70b-tp8"
    if llama:
        eng, cfg, wl = make_llama(a, hw, world, rank, dak, cal_kw)
    else:
        layers = a.layers or 48
        cfg = OPT_30B if layers == 48 else OPTConfig(n_layers=layers)
        eng = DakOPT(cfg, a.batch, a.context, hw, mode=dak.PLAN_BALANCED, y_req=0, pdl=not a.no_pdl,
                     congestion_control=not a.no_cc, l2_prefetch=int(a.l2_prefetch_mb * (1 << 20)),
                     evict_first=not a.no_evict_first, fuse_norm=not a.no_fuse_norm,
                     seed=1234 + rank, chunk_pages=a.chunk_pages, **cal_kw)
        if a.ratio is not None:  # forced global ratio: EXACT mode at y_req = R * sum C_i
            tot = sum(o["total_bytes"] for o in eng.plan_ops)
            eng.close()
            eng = DakOPT(cfg, a.batch, a.context, hw, mode=dak.PLAN_EXACT, y_req=int(a.ratio * tot), pdl=not a.no_pdl,
                         congestion_control=not a.no_cc, l2_prefetch=int(a.l2_prefetch_mb * (1 << 20)),
                         evict_first=not a.no_evict_first, fuse_norm=not a.no_fuse_norm,
                         seed=1234 + rank, chunk_pages=a.chunk_pages, **cal_kw)
    nb = eng.bytes_per_step()
    stream = torch.cuda.Stream()
    g = eng.capture(stream)
    for _ in range(a.warmup):
        g.replay()
    torch.cuda.synchronize()

    # ---------------- device-timed region: K graph replays (inputs 60 GB >> 126 MB L2: no flush)
    sampler = ClockSampler(local, os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp",
                                               f"clocks_rank{rank}.csv"))
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(a.steps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    t = e0.elapsed_time(e1) / 1e3
    t_max = reduce_max(t, world)
    # per-rank rates (each GPU reads its own host shard over its own link)
    mine = dict(rank=rank, ms_per_step=round(t / a.steps * 1e3, 4), host_link_gbs=round(nb["host"] * a.steps / t / 1e9, 2),
                hbm_gbs=round(nb["hbm"] * a.steps / t / 1e9, 1))
    per_rank = [mine]
    if world > 1:
        import torch.distributed as dist
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    step_s = t_max / a.steps
    value = nb["total"] * world * a.steps / t_max / 1e9
    reqs = eng.B if llama else eng.B * world  # TP: one batch over all ranks; replicas: one per rank
    tok_s = reqs * a.steps / t_max

    # ---------------- end to end through the public API with host buffers
    tok_host = torch.zeros(eng.B, dtype=torch.int32).pin_memory()
    logits_host = torch.empty(eng.B, eng.logits.shape[1], dtype=torch.bfloat16).pin_memory()
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for i in range(a.steps):
            tok_host.fill_(i % cfg.vocab)
            eng.tokens.copy_(tok_host, non_blocking=True)
            g.replay()
            logits_host.copy_(eng.logits, non_blocking=True)
        e1.record(stream)
    torch.cuda.synchronize()
    te = reduce_max(e0.elapsed_time(e1) / 1e3, world)
    e2e = dict(value=round(nb["total"] * world * a.steps / te / 1e9, 2), unit="GB/s",
               tokens_per_s=round(reqs * a.steps / te, 2),
               h2d_bytes_per_step=tok_host.numel() * 4, d2h_bytes_per_step=logits_host.numel() * 2)

    # ---------------- roofline of the dominant kernel (dak_linear), measured INSIDE the step
    # One step is captured with the library's globaltimer launch trace on (dak_trace_enable) and
    # replayed; each launch is charged the time it adds to the step's timeline (its last CTA's end
    # minus the previous launch's last end: with PDL the launches overlap, so this partitions the
    # step without double counting). dak_linear's share = the sum over its launches, in the exact
    # variants the step runs (fused pre-norm, SwiGLU operand, residual epilogues, attention between).
    # The replays are bracketed by CUDA events on the launching stream (traced vs untraced step time).
    prof = in_step_profile(eng, stream, torch, dak, reps=5)
    ops = list(eng.linear_ops())
    lin_bytes = sum(op.M * op.K * 2 + eng.B * (op.K + op.M) * 2 for op in ops)  # algorithmic, per step
    lin_time = prof["linear_s"]
    lin_achieved = lin_bytes / lin_time / 1e9
    # peak: the split roofline at the linears' own host ratio, EB(r) = 1 / max((1 - r)/B_g, r/B_l)
    # (= B_g + B_l at r*, B_l / r for a capacity-forced, link-bound plan)
    r_lin = sum(op.h * op.K * 2 for op in ops) / max(1, sum(op.M * op.K * 2 for op in ops))
    peak = 1.0 / max((1.0 - r_lin) / hbm_gbs, r_lin / link_gbs) if r_lin > 0 else hbm_gbs
    # traffic: DRAM read+write bytes per dak_linear launch of THIS workload from the committed ncu
    # capture (profiles/r*/linear_traffic_<workload>.json, tools/summarize_profiles.py)
    wl_name = wl["workload"] if llama else "opt-30b-decode-b%d-ctx%d" % (eng.B, a.context)
    traffic, tr_src = None, None
    tr_files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "linear_traffic_%s.json" % wl_name)))
    if tr_files:
        tr = json.load(open(tr_files[-1]))
        traffic, tr_src = tr["dram_bytes_per_launch"], os.path.relpath(tr_files[-1], ROOT)
    roofline = dict(bound="hbm", achieved=round(lin_achieved, 1), peak=round(peak, 1), unit="GB/s",
                    frac=round(lin_achieved / peak, 4), traffic=traffic,
                    algorithmic_bytes_per_launch=round(lin_bytes / len(ops)),
                    launches_per_step=len(ops), avg_launch_us=round(lin_time / len(ops) * 1e6, 3),
                    traffic_source=tr_src,
                    kernel="dak_linear (split GEMV / skinny GEMM), timed inside the captured decode step: per-launch "
                           "timeline increments from the library's globaltimer trace, summed over the step's %d "
                           "linear launches" % len(ops),
                    peak_source="EB(r) = 1/max((1-r)/B_g, r/B_l) at the linears' host ratio r = %.5f: B_g = %s HBM copy "
                                "%.1f GB/s (MEASURED_PEAKS.json hbm_gbs), B_l = measured host link %.1f GB/s"
                                % (r_lin, peak_src, hbm_gbs, link_gbs),
                    frac_of_copy_plus_link=round(lin_achieved / (hbm_gbs + link_gbs), 4),
                    # read-only streams exceed the copy figure: the calibrated bulk-read ring peak
                    # (profiles/r01/calib_loadpath.jsonl, 148 SMs x 4 x 32 KB) as a second denominator
                    read_peak=round(READ_PEAK_GBS + link_gbs, 1),
                    frac_of_read_peak=round(lin_achieved / (READ_PEAK_GBS + link_gbs), 4),
                    kernel_time_share_of_step=round(lin_time / prof["traced_step_s"], 4),
                    traced_step_ms=round(prof["traced_step_s"] * 1e3, 4),
                    untraced_step_ms=round(step_s * 1e3, 4),
                    share_by_kind={k: round(v / prof["traced_step_s"], 4) for k, v in prof["by_kind_s"].items()})
    # the split roofline at the step's host ratio r: EB(r) = 1 / max((1 - r)/B_g, r/B_l),
    # = B_g + B_l at r* and B_l / r above it (a capacity-forced step is link-bound)
    r_step = nb["host"] / nb["total"]
    eb_r = 1.0 / max((1.0 - r_step) / hbm_gbs, r_step / link_gbs)
    roofline.update(split_roofline_gbs=round(eb_r, 1), split_roofline_r=round(r_step, 5),
                    step_frac_of_split_roofline=round(value / world / eb_r, 4))

    line = dict(metric=METRIC, value=round(value, 2), unit="GB/s", n_gpus=world, steps=a.steps, warmup=a.warmup,
                ms_per_step=round(step_s * 1e3, 4), higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="bf16", data="synthetic (random-init %s weights and KV)" % cfg.name,
                config=(dict(wl, host_bytes_per_step=nb["host"], hbm_bytes_per_step=nb["hbm"],
                             host_ratio=round(nb["host"] / nb["total"], 5), pdl=not a.no_pdl,
                             congestion_control=not a.no_cc, execution="per-op kernels (dak_layer, PDL, CUDA graph)")
                        if llama else dict(workload="opt-30b-decode-b%d-ctx%d" % (eng.B, a.context), model_shape="OPT-30B",
                            batch=eng.B, context=a.context, layers=cfg.n_layers,
                            plan="BALANCED" if a.ratio is None else "EXACT R=%.4f" % a.ratio,
                            host_bytes_per_step=nb["host"], hbm_bytes_per_step=nb["hbm"],
                            host_ratio=round(nb["host"] / nb["total"], 5),
                            l2="inputs (60 GB of weights) >> 126 MB L2; no flush",
                            pdl=not a.no_pdl, congestion_control=not a.no_cc,
                            planner_rates_gbs=dict(hbm=round(hw.hbm_bps / 1e9, 1), link=round(hw.link_bps / 1e9, 2),
                                                   host_latency_us=a.plan_host_latency_us, source=plan_src),
                            execution="per-op kernels (dak_layer, PDL, CUDA graph)",
                            parallelism="dp%d replicas (weak scaling, no collective)" % world)),
                tokens_per_s=round(tok_s, 2), roofline=roofline, e2e=e2e, clocks=clocks, per_rank=per_rank,
                **({"calibration": dict(cal, hbm_gbs=round(cal["hbm_bps"] / 1e9, 1), link_gbs=round(cal["link_bps"] / 1e9, 2),
                                        host_latency_us=round(cal["host_latency_s"] * 1e6, 3))} if cal else {}),
                **({"tokens_per_s_full_model_extrapolated": round(tok_s * cfg.n_layers / 80, 2)}
                   if llama and cfg.n_layers != 80 else {}),
                gpu_launches=eng.kernels_per_step() * a.steps)
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not llama:
        v, dt, nbytes, threads, reps = oracle_sample(eng.B)
        line["cpu_baseline"] = dict(value=round(v, 3), unit="GB/s", cores=threads, kind="oracle",
                                    sample="OPT-30B layer-0 q/k/v/o/fc1/fc2 float64 oracle linears (N=%d) + 56-head "
                                           "decode attention over 64 tokens, x%d (%.1f s)" % (eng.B, reps, dt))
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if getattr(eng, "comm_handle", None):
        dak.comm_destroy(eng.comm_handle)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
