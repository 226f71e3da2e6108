"""DAK decode engine for Llama-family models under tensor parallelism (BASELINE configs[2]:
Llama-3-70B, TP8 over 8 x B200, weights + KV larger than HBM), built on the C ABI.

One instance = one tensor-parallel rank (one GPU): it owns its Megatron shard (tp.py) of every
weight and its kv heads' KV cache, plans per-op host ratios for ITS op list with the greedy
planner (each GPU reads its own host link), places and packs the tiers, and enqueues
the decode step: embed (+ row statistics) -> layers (dak_layer, DAK_MODEL_LLAMA: RMSNorm fused into
q/k/v and [gate; up], rotary + KV append, split attention, o / down with residual, NCCL
all-reduce of the row-parallel partials when tp_size > 1) -> LM head shard (final RMSNorm fused).
torch is used for device memory, streams and graphs only; this module never imports the oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import dak, tp
from .engine import HW, LinearOp, _bf16_rand


@dataclass
class LlamaConfig:
    n_layers: int = 80
    hidden: int = 8192
    n_heads: int = 64
    n_kv_heads: int = 8
    ffn: int = 28672
    vocab: int = 128256
    head_dim: int = 128
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    name: str = "llama-3-70b"


LLAMA3_70B = LlamaConfig()


class DakLlama:
    """Decode step of one tensor-parallel rank over HBM + pinned host memory at planned ratios."""

    def __init__(self, cfg: LlamaConfig, batch: int, context: int, hw: HW, tp_rank: int = 0, tp_size: int = 1,
                 comm=None, mode: int = dak.PLAN_BALANCED, y_req: int = 0, unit_rows: int = 16, page_size: int = 64,
                 chunk_pages: int = 0, seed: int = 0, pdl: bool = True, congestion_control: bool = True,
                 weights: dict | None = None, n_cta_host: int = 2, fuse_norm: bool | None = None):
        self.cfg, self.B, self.context, self.hw = cfg, batch, context, hw
        self.rank, self.world, self.comm = tp_rank, tp_size, comm
        # operand transforms fused into the linears only at small batch: above 16 columns every CTA
        # would re-normalise / re-activate the whole operand (measured 3-8x slower than one kernel)
        self.fuse_norm = (batch <= 16) if fuse_norm is None else bool(fuse_norm)
        self.dims = tp.local_dims(cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.vocab, tp_size)
        self.page, self.chunk_pages, self.unit_rows = page_size, chunk_pages, unit_rows
        if not chunk_pages:  # split-KV chunk: about one (request, kv head, chunk) unit per two warp slots (measured best)
            pages = -(-context // page_size)
            units_1 = batch * (cfg.n_kv_heads // tp_size) * pages
            self.chunk_pages = max(1, min(16, units_1 // (148 * 4)))
        self.pdl = int(pdl)
        self.n_cta_host = n_cta_host
        self.launch = dict(pdl=self.pdl, congestion_control=int(congestion_control), n_cta_host=n_cta_host)
        self.sms = dak.device_sms()
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed + 7919 * tp_rank)
        self._host_blocks = []
        c, d = cfg, cfg.head_dim
        nh, nkv, F = self.dims["n_heads"], self.dims["n_kv"], self.dims["ffn"]
        self.layers = []
        for i in range(c.n_layers):
            self.layers.append(dict(qkv=LinearOp(f"L{i}.qkv", (nh + 2 * nkv) * d, c.hidden),
                                    o=LinearOp(f"L{i}.o", c.hidden, nh * d),
                                    up=LinearOp(f"L{i}.gate_up", 2 * F, c.hidden),
                                    down=LinearOp(f"L{i}.down", c.hidden, F)))
        self.head = LinearOp("lm_head", self.dims["vocab"], c.hidden)
        self.pages_per_req = -(-context // page_size)
        self.chunks_per_req = -(-self.pages_per_req // self.chunk_pages)
        self.plan = self._plan(mode, y_req)
        self._allocate(weights)
        self._kv()
        self.graph = None

    # ------------------------------------------------------------------ planning
    def linear_ops(self):
        for L in self.layers:
            yield from (L["qkv"], L["o"], L["up"], L["down"])
        yield self.head

    def _plan(self, mode, y_req):
        c, B = self.cfg, self.B
        ops = []
        for op in self.linear_ops():
            ops.append(dict(kind="linear", n_units=-(-op.M // self.unit_rows), unit_bytes=self.unit_rows * op.K * 2,
                            total_bytes=op.bytes, T=2.0 * B * op.M * op.K / self.hw.peak_flops))
        tok_bytes = 2 * self.dims["n_kv"] * c.head_dim * 2
        for _ in range(c.n_layers):
            C_att = tok_bytes * B * self.context
            n_units = B * self.chunks_per_req
            ops.append(dict(kind="attention", n_units=n_units, unit_bytes=-(-C_att // n_units), total_bytes=C_att,
                            T=4.0 * B * self.context * self.dims["n_heads"] * c.head_dim / self.hw.peak_flops))
        self.plan_ops = ops
        plan, self.objective = dak.plan_ratios(self.hw.as_dict(), ops, y_req, mode)
        for i, op in enumerate(self.linear_ops()):
            op.h = min(op.M, plan[i]["host_units"] * self.unit_rows)
            n_host = min(self.n_cta_host, op.h) if op.h > 0 else 0
            rows = max(-(-op.h // max(n_host, 1)) if op.h else 0, -(-(op.M - op.h) // (self.sms - n_host)))
            # KC = 64 above 16 batch columns: the tcgen05 path (canonical SWIZZLE_128B operands)
            op.kc = 64 if self.B > 16 else dak.step_choose_kc(rows, op.K)
        n_lin = 4 * c.n_layers + 1
        self.attn_host_chunks = [plan[n_lin + l]["host_units"] for l in range(c.n_layers)]
        return plan

    # ------------------------------------------------------------------ placement + packing
    def _alloc_host(self, nbytes):
        hp, dp = dak.host_alloc(max(nbytes, 16))
        self._host_blocks.append(hp)
        return hp, dp

    def _fill_linear(self, op: LinearOp, W):
        M, K, h = op.M, op.K, op.h
        if h < M:
            op.hbm = torch.empty((M - h) * K, dtype=torch.bfloat16, device="cuda")
            if W is None:
                op.hbm.copy_(_bf16_rand(((M - h) * K,), 1.0 / math.sqrt(K), self.gen))
            else:
                dak.pack_linear(W[h:].contiguous(), M - h, K, op.kc, op.hbm)
        if h > 0:
            op.host = self._alloc_host(h * K * 2)
            src = W[:h].contiguous() if W is not None else _bf16_rand((h, K), 1.0 / math.sqrt(K), self.gen)
            dak.pack_linear(src, h, K, op.kc, op.host[1])

    def _allocate(self, weights):
        """weights: FULL logical parameters as device bf16 tensors (names as oracle/layer.py), sharded
        here for this rank; None -> random weights of the shard's shapes."""
        c, dev = self.cfg, "cuda"
        loc = None
        if weights:
            loc = tp.shard_llama(weights, self.rank, self.world, c.n_heads, c.n_kv_heads, c.head_dim)
        for i, L in enumerate(self.layers):
            for key, op in L.items():
                if loc is None:
                    W = None
                elif key == "up":
                    W = torch.cat([loc[f"L{i}.gate"], loc[f"L{i}.up"]], dim=0)
                elif key == "qkv":
                    W = torch.cat([loc[f"L{i}.q"], loc[f"L{i}.k"], loc[f"L{i}.v"]], dim=0)
                else:
                    W = loc[f"L{i}.{key}"]
                self._fill_linear(op, W)
            for n in ("ln1_w", "ln2_w"):
                L[n] = loc[f"L{i}.{n}"].contiguous() if loc else torch.ones(c.hidden, dtype=torch.bfloat16, device=dev)
        self.tok_emb = loc["embed"].contiguous() if loc else _bf16_rand((c.vocab, c.hidden), 0.02, self.gen)
        self._fill_linear(self.head, loc["lm_head"] if loc else None)
        self.lnf_w = loc["lnf_w"].contiguous() if loc else torch.ones(c.hidden, dtype=torch.bfloat16, device=dev)
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ KV cache (paged)
    def _kv(self):
        c, B = self.cfg, self.B
        ppr, cp = self.pages_per_req, self.chunk_pages
        nkv = self.dims["n_kv"]
        page_elems = nkv * self.page * c.head_dim
        self.block_tables, self.kv = [], []
        for l in range(c.n_layers):
            hu = self.attn_host_chunks[l]
            host_pages = [min(ppr, (hu // B + (1 if b < hu % B else 0)) * cp) for b in range(B)]
            Ph = sum(host_pages)
            Pg = B * ppr - Ph
            bt = np.zeros((B, ppr), dtype=np.int64)
            ih = ig = 0
            for b in range(B):
                for p in range(ppr):
                    if p < host_pages[b]:
                        bt[b, p] = ih | 0x80000000
                        ih += 1
                    else:
                        bt[b, p] = ig
                        ig += 1
            kg = torch.zeros(max(Pg, 1) * page_elems, dtype=torch.bfloat16, device="cuda")
            vg = torch.zeros_like(kg)
            kh = self._alloc_host(max(Ph, 1) * page_elems * 2)
            vh = self._alloc_host(max(Ph, 1) * page_elems * 2)
            for hp in (kh, vh):
                n = max(Ph, 1) * page_elems
                np.ctypeslib.as_array((__import__("ctypes").c_uint16 * n).from_address(hp[0]))[:] = 0
            kg.copy_(_bf16_rand(kg.shape, 1.0, self.gen))
            vg.copy_(_bf16_rand(vg.shape, 1.0, self.gen))
            self.kv.append((kg, vg, kh, vh, Ph, Pg))
            self.block_tables.append(torch.from_numpy((bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda())
        self.positions = torch.full((B,), self.context - 1, dtype=torch.int32, device="cuda")
        self.seq_lens = self.positions + 1
        self.tokens = torch.zeros((B,), dtype=torch.int32, device="cuda")
        self.x = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.hnorm = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.logits = torch.empty((B, self.dims["vocab"]), dtype=torch.bfloat16, device="cuda")
        self.layer_args = [self._layer_args(l) for l in range(c.n_layers)]
        self.scratch = torch.empty(dak.layer_scratch_size(self.layer_args[0]), dtype=torch.uint8, device="cuda")
        self.stats = torch.zeros((1024, B, 4), dtype=torch.float32, device="cuda")
        parts = 1
        for a in self.layer_args:
            a.scratch, a.scratch_bytes = self.scratch.data_ptr(), self.scratch.numel()
            a.stats_in, a.stats_in_parts, a.stats_out = self.stats.data_ptr(), parts, self.stats.data_ptr()
            parts = dak.layer_stats_parts(a)
        self.head_stats_parts = parts

    def load_kv(self, K_cache, V_cache):
        """K_cache[l][b] = [L_b, Hkv_local, d] bf16 bits of this rank's kv heads for the cached tokens
        (already rotated), written into the tier pools named by the block table (DAK-PG)."""
        d, nkv, page = self.cfg.head_dim, self.dims["n_kv"], self.page
        for l, (kg, vg, kh, vh, Ph, Pg) in enumerate(self.kv):
            bt = self.block_tables[l].cpu().numpy().view(np.uint32)
            pools = {}
            for name, src in (("k", K_cache[l]), ("v", V_cache[l])):
                lg = np.zeros((max(Pg, 1), nkv, page, d), np.uint16)
                lh = np.zeros((max(Ph, 1), nkv, page, d), np.uint16)
                for b in range(self.B):
                    arr = np.asarray(src[b])
                    for t0 in range(0, arr.shape[0], page):
                        e = int(bt[b, t0 // page])
                        pool = lh if e & 0x80000000 else lg
                        blk = arr[t0:t0 + page]
                        pool[e & 0x7FFFFFFF, :, :blk.shape[0]] = blk.transpose(1, 0, 2)
                pools[name] = (lg, lh)
            for (lg, lh), dg, dh in ((pools["k"], kg, kh), (pools["v"], vg, vh)):
                dak.pack_kv_pages(torch.from_numpy(lg.view(np.int16)).cuda(), lg.shape[0] * nkv, page, d, dg)
                dak.pack_kv_pages(torch.from_numpy(lh.view(np.int16)).cuda(), lh.shape[0] * nkv, page, d, dh[1])
                torch.cuda.synchronize()

    def _layer_args(self, l):
        c, L = self.cfg, self.layers[l]
        kg, vg, kh, vh, Ph, Pg = self.kv[l]
        a = dak.dak_layer_args()
        a.model, a.B, a.hidden = dak.MODEL_LLAMA, self.B, c.hidden
        a.n_heads, a.n_kv_heads, a.head_dim, a.ffn = self.dims["n_heads"], self.dims["n_kv"], c.head_dim, self.dims["ffn"]
        a.ln_eps, a.rope_theta = c.rms_eps, c.rope_theta
        a.split_qkv = 0
        a.qkv = L["qkv"].weight()
        a.o, a.up, a.down = L["o"].weight(), L["up"].weight(), L["down"].weight()
        a.ln1_w, a.ln2_w = L["ln1_w"].data_ptr(), L["ln2_w"].data_ptr()
        a.x = self.x.data_ptr()
        a.k_hbm, a.v_hbm = kg.data_ptr(), vg.data_ptr()
        a.k_host, a.v_host = kh[1], vh[1]
        a.block_table, a.positions, a.seq_lens = (self.block_tables[l].data_ptr(), self.positions.data_ptr(),
                                                  self.seq_lens.data_ptr())
        a.page_size, a.max_pages, a.chunk_pages = self.page, self.pages_per_req, self.chunk_pages
        a.tp_rank, a.tp_size, a.comm = self.rank, self.world, self.comm
        a.fuse_norm = int(self.fuse_norm)
        if not self.fuse_norm and self.comm:  # the down combine writes the next layer's RMSNorm 1
            a.x_prenormed = int(l > 0)
            a.next_ln_w = self.layers[l + 1]["ln1_w"].data_ptr() if l + 1 < c.n_layers else None
        a.cfg = dak.launch_cfg(**self.launch)
        # attention host CTAs: ~one per 8 host units (units = chunks x kv heads; one unit per warp)
        n_kvh = getattr(self, "dims", {}).get("n_kv", None) or c.n_kv_heads
        host_units = self.attn_host_chunks[l] * n_kvh
        a.attn_cfg = dak.launch_cfg(**dict(self.launch, n_cta_host=dak.attention_host_ctas(host_units)))
        return a

    # ------------------------------------------------------------------ the decode step (hot path)
    def enqueue_step(self, stream=None):
        c = self.cfg
        dak.embed(self.tokens, None, self.tok_emb, None, self.B, c.hidden, 0, self.x, pdl=self.pdl, stream=stream,
                  stats_out=self.stats if self.fuse_norm else None)
        for a in self.layer_args:
            dak.layer(a, stream)
        hw = self.head.host[1] if self.head.host else None
        if self.fuse_norm:  # final RMSNorm fused into the LM head
            ha = dak.linear_args(hw, self.head.hbm, self.head.M, self.head.K, self.head.h, self.head.kc, self.B, self.x,
                                 self.logits, cfg=self.launch, ln_w=self.lnf_w, ln_stats=self.stats,
                                 ln_parts=self.head_stats_parts, ln_rms=1, ln_eps=c.rms_eps)
        else:
            dak.rmsnorm(self.x, self.lnf_w, self.hnorm, self.B, c.hidden, c.rms_eps, pdl=self.pdl, stream=stream)
            ha = dak.linear_args(hw, self.head.hbm, self.head.M, self.head.K, self.head.h, self.head.kc, self.B,
                                 self.hnorm, self.logits, cfg=self.launch)
        if self.B > 16:  # tcgen05 split-K partials for the head
            need = dak.linear_workspace_size(ha)
            if need:
                if getattr(self, "head_ws", None) is None or self.head_ws.numel() < need:
                    self.head_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
                ha.workspace, ha.workspace_bytes = self.head_ws.data_ptr(), self.head_ws.numel()
        dak.linear(ha, stream)

    def _reduce_launches(self, op) -> int:
        """1 when this linear splits K on the tcgen05 path (one split-K reduce kernel), else 0."""
        if self.B <= 16:
            return 0
        w = op.weight()
        la = dak.linear_args(op.host[1] if op.host else None, op.hbm, op.M, op.K, op.h, op.kc, self.B, 16, 16,
                             cfg=dict(self.launch, n_cta_host=w.n_cta_host or self.launch["n_cta_host"]))
        la.workspace, la.workspace_bytes = 256, 1 << 40  # query only: the plan splits K when workspace is given
        return int(dak.linear_query(la)["ksplit"] > 1)

    def kernels_per_step(self) -> int:
        """Kernels of this library per decode step (NCCL's own kernels not counted)."""
        L = self.cfg.n_layers
        per_layer = (6 + (1 if self.chunks_per_req > 1 else 0)  # qkv, rope+append, attention, o, up, down (+combine)
                     + (2 if self.comm else 0)  # residual (+ RMSNorm) kernels after the all-reduces
                     + (0 if self.fuse_norm else (1 if self.comm else 3)))  # silu*up (+ RMSNorm 1, RMSNorm 2)
        n = 1 + per_layer * L + (1 if self.fuse_norm else 2)  # embed ... (final RMSNorm +) head
        if not self.fuse_norm and self.comm:
            n += 1  # RMSNorm 1 of layer 0 (later layers get it from the previous combine)
        # split-K reduces: qkv's and [gate; up]'s are fused into the rotary / silu kernels when unfused
        ops = list(self.linear_ops())
        for i, op in enumerate(ops):
            fused_reduce = not self.fuse_norm and i < 4 * L and i % 4 in (0, 2)
            n += 0 if fused_reduce else self._reduce_launches(op)
        return n

    def capture(self, stream: torch.cuda.Stream):
        with torch.cuda.stream(stream):
            self.enqueue_step(stream)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self.enqueue_step(stream)
        self.graph = g
        return g

    def bytes_per_step(self) -> dict:
        hbm = host = 0
        for op in self.linear_ops():
            hbm += (op.M - op.h) * op.K * 2
            host += op.h * op.K * 2
        tok = 2 * self.dims["n_kv"] * self.cfg.head_dim * 2
        for (kg, vg, kh, vh, Ph, Pg) in self.kv:
            hp = min(Ph * self.page, self.B * self.context)
            host += tok * hp
            hbm += tok * (self.B * self.context - hp)
        return dict(hbm=hbm, host=host, total=hbm + host)

    def close(self):
        for hp in self._host_blocks:
            try:
                dak.host_free(hp)
            except Exception:
                pass
        self._host_blocks = []
