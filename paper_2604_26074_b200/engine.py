"""DAK decode engine for OPT-family models (PAPER §4), built on the C ABI.

Setup (once): operator list -> dak_plan_ratios (greedy per-op ratios) -> byte
placement (host = leading rows / oldest KV chunks) -> DAK-KC / DAK-PG packing into HBM
and pinned mapped host memory -> one decode step captured in a CUDA graph.
Step (hot path): embed -> 48 x dak_layer -> LayerNorm -> LM head, every weight and KV page
streamed by the library's split-source kernels. torch is used only for device memory, streams
and graphs. This module never imports the CPU oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import dak


@dataclass
class OPTConfig:
    n_layers: int = 48
    hidden: int = 7168
    n_heads: int = 56
    ffn: int = 28672
    vocab: int = 50272
    max_pos: int = 2048
    head_dim: int = 128
    name: str = "opt-30b"

    @property
    def n_kv_heads(self) -> int:
        return self.n_heads


OPT_30B = OPTConfig()


@dataclass
class HW:
    """Planner machine model (bytes/s). B_h = min(link, host DRAM) (P:L216 footnote)."""
    hbm_bps: float
    link_bps: float
    host_dram_bps: float = 0.0
    peak_flops: float = 1.3554e15
    host_latency_s: float = 0.0  # latency-aware planner extension (dak_hw.host_latency_s)

    def as_dict(self):
        return dict(hbm_bps=self.hbm_bps, link_bps=self.link_bps,
                    host_dram_bps=self.host_dram_bps or self.link_bps, host_capacity_bytes=-1,
                    host_latency_s=self.host_latency_s)


@dataclass
class LinearOp:
    name: str
    M: int
    K: int
    h: int = 0
    kc: int = 64
    hbm: torch.Tensor | None = None
    host: tuple | None = None  # (host_ptr, dev_ptr)
    bias: torch.Tensor | None = None

    @property
    def bytes(self) -> int:
        return self.M * self.K * 2

    def weight(self) -> dak.dak_weight:
        return dak.weight(self.host[1] if self.host else None, self.hbm, self.h, self.kc, self.bias)


def _bf16_rand(shape, std, gen):
    return (torch.randn(shape, device="cuda", generator=gen, dtype=torch.float32) * std).to(torch.bfloat16)


class DakOPT:
    """OPT decode step over HBM + pinned host memory at per-op planned ratios."""

    def __init__(self, cfg: OPTConfig, batch: int, context: int, hw: HW, mode: int = dak.PLAN_BALANCED,
                 y_req: int = 0, unit_rows: int = 16, page_size: int = 64, chunk_pages: int = 0, seed: int = 0,
                 pdl: bool = True, congestion_control: bool = True, weights: dict | None = None,
                 host_override: dict | None = None, n_cta_host: int = 2, l2_prefetch: int = 0,
                 evict_first: bool = True, fuse_norm: bool = True, fused_qkv: bool = True,
                 max_context: int | None = None):
        self.cfg, self.B, self.context, self.hw = cfg, batch, context, hw
        self.page, self.chunk_pages, self.unit_rows = page_size, chunk_pages, unit_rows
        if not chunk_pages:  # split-KV chunk: about one (request, kv head, chunk) unit per two warp slots (measured best)
            pages = -(-max(context, max_context or 0) // page_size)
            units_1 = batch * cfg.n_kv_heads * pages
            self.chunk_pages = max(1, min(16, units_1 // (148 * 4)))
        self.pdl = int(pdl)
        self.n_cta_host = n_cta_host
        self.launch = dict(pdl=self.pdl, congestion_control=int(congestion_control), n_cta_host=n_cta_host,
                           l2_policy=0 if evict_first else 1)
        self.l2_prefetch = int(l2_prefetch)
        self.fuse_norm = bool(fuse_norm)
        # one [q; k; v] projection per layer (one launch reading x once); the persistent step and
        # the paper's op list use the three projections separately
        self.fused_qkv = bool(fused_qkv)
        self.sms = dak.device_sms()
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed)
        self._host_blocks = []
        c = cfg
        self.layers = []
        for i in range(c.n_layers):
            if self.fused_qkv:
                L = dict(qkv=LinearOp(f"L{i}.qkv", (c.n_heads + 2 * c.n_kv_heads) * c.head_dim, c.hidden))
            else:  # q/k/v separate, as the paper's op list (P:L981 footnote)
                L = dict(q=LinearOp(f"L{i}.q", c.n_heads * c.head_dim, c.hidden),
                         k=LinearOp(f"L{i}.k", c.n_kv_heads * c.head_dim, c.hidden),
                         v=LinearOp(f"L{i}.v", c.n_kv_heads * c.head_dim, c.hidden))
            L.update(o=LinearOp(f"L{i}.o", c.hidden, c.n_heads * c.head_dim),
                     up=LinearOp(f"L{i}.fc1", c.ffn, c.hidden),
                     down=LinearOp(f"L{i}.fc2", c.hidden, c.ffn))
            self.layers.append(L)
        self.head = LinearOp("head", c.vocab, c.hidden)
        # KV pages per request cover max_context tokens: decode steps append beyond the prompt
        self.max_context = max(context, max_context or context)
        self.pages_per_req = -(-self.max_context // page_size)
        self.chunks_per_req = -(-self.pages_per_req // self.chunk_pages)
        self.plan = self._plan(mode, y_req, host_override)
        self._allocate(weights)
        self._kv()
        self.graph = None

    # ------------------------------------------------------------------ planning
    def linear_ops(self):
        for L in self.layers:
            if self.fused_qkv:
                yield from (L["qkv"], L["o"], L["up"], L["down"])
            else:
                yield from (L["q"], L["k"], L["v"], L["o"], L["up"], L["down"])
        yield self.head

    def kv_bytes_per_layer(self) -> int:
        c = self.cfg
        return 2 * c.n_kv_heads * c.head_dim * 2 * self.B * self.context

    def _plan(self, mode, y_req, host_override):
        c, B = self.cfg, self.B
        ops = []
        for op in self.linear_ops():
            flops = 2.0 * B * op.M * op.K
            ops.append(dict(kind="linear", n_units=-(-op.M // self.unit_rows), unit_bytes=self.unit_rows * op.K * 2,
                            total_bytes=op.bytes, T=flops / self.hw.peak_flops))
        tok_bytes = 2 * c.n_kv_heads * c.head_dim * 2
        chunk_tok = self.chunk_pages * self.page
        for _ in range(c.n_layers):
            C_att = tok_bytes * B * self.context
            n_units = B * self.chunks_per_req
            # every request's last chunk may be short: plan with the mean unit (ceil(C/n)), which
            # keeps (n-1)u < C <= nu; placement then takes whole chunks, oldest first (DESIGN R15)
            unit = -(-C_att // n_units)
            flops = 4.0 * B * self.context * c.n_heads * c.head_dim
            ops.append(dict(kind="attention", n_units=n_units, unit_bytes=unit, total_bytes=C_att,
                            T=flops / self.hw.peak_flops))
        self.plan_ops = ops
        plan, obj = dak.plan_ratios(self.hw.as_dict(), ops, y_req, mode)
        self.objective = obj
        i = 0
        for op in self.linear_ops():
            op.h = min(op.M, plan[i]["host_units"] * self.unit_rows)
            if host_override and op.name.split(".")[-1] in host_override:
                op.h = host_override[op.name.split(".")[-1]]
            # one KC for both execution paths: the persistent step's slot constraint (<= 256)
            n_host = min(self.n_cta_host, op.h) if op.h > 0 else 0
            rows = max(-(-op.h // max(n_host, 1)) if op.h else 0, -(-(op.M - op.h) // (self.sms - n_host)))
            # KC = 64 above 16 batch columns: the tcgen05 path (canonical SWIZZLE_128B operands)
            op.kc = 64 if self.B > 16 else dak.step_choose_kc(rows, op.K)
            i += 1
        self.attn_host_chunks = [plan[i + l]["host_units"] for l in range(c.n_layers)]
        return plan

    # ------------------------------------------------------------------ placement + packing
    def _alloc_host(self, nbytes):
        hp, dp = dak.host_alloc(max(nbytes, 16))
        self._host_blocks.append(hp)
        return hp, dp

    def _fill_linear(self, op: LinearOp, W: torch.Tensor | None):
        """W: logical [M, K] bf16 on device (or None: random N(0, 1/K) drawn in packed order)."""
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
        c = self.cfg
        dev = "cuda"
        if weights:  # a fused [q;k;v] weight may be given: split it into the three projections
            weights = dict(weights)
            for i in range(c.n_layers):
                if self.fused_qkv and f"L{i}.qkv" not in weights:
                    weights[f"L{i}.qkv"] = torch.cat([weights.pop(f"L{i}.{k}") for k in ("q", "k", "v")])
                    weights[f"L{i}.qkv.b"] = torch.cat([weights.pop(f"L{i}.{k}.b") for k in ("q", "k", "v")])
                if not self.fused_qkv and f"L{i}.qkv" in weights:
                    Wf, bf = weights.pop(f"L{i}.qkv"), weights.pop(f"L{i}.qkv.b")
                    r0 = 0
                    for key in ("q", "k", "v"):
                        M = self.layers[i][key].M
                        weights[f"L{i}.{key}"], weights[f"L{i}.{key}.b"] = Wf[r0:r0 + M], bf[r0:r0 + M]
                        r0 += M
        for i, L in enumerate(self.layers):
            for key, op in list(L.items()):
                W = weights[f"L{i}.{key}"] if weights else None
                self._fill_linear(op, W)
                op.bias = weights[f"L{i}.{key}.b"].contiguous() if weights else _bf16_rand((op.M,), 0.02, self.gen)
            L["ln1_w"] = weights[f"L{i}.ln1_w"] if weights else torch.ones(c.hidden, dtype=torch.bfloat16, device=dev)
            L["ln1_b"] = weights[f"L{i}.ln1_b"] if weights else torch.zeros(c.hidden, dtype=torch.bfloat16, device=dev)
            L["ln2_w"] = weights[f"L{i}.ln2_w"] if weights else torch.ones(c.hidden, dtype=torch.bfloat16, device=dev)
            L["ln2_b"] = weights[f"L{i}.ln2_b"] if weights else torch.zeros(c.hidden, dtype=torch.bfloat16, device=dev)
        emb = weights["embed"] if weights else _bf16_rand((c.vocab, c.hidden), 0.02, self.gen)
        self.tok_emb = emb
        self.pos_emb = weights["pos"] if weights else _bf16_rand((c.max_pos + 2, c.hidden), 0.02, self.gen)
        self._fill_linear(self.head, emb)  # OPT ties the LM head to the token embedding
        self.lnf_w = weights["lnf_w"] if weights else torch.ones(c.hidden, dtype=torch.bfloat16, device=dev)
        self.lnf_b = weights["lnf_b"] if weights else torch.zeros(c.hidden, dtype=torch.bfloat16, device=dev)
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ KV cache (paged)
    def _kv(self):
        c, B = self.cfg, self.B
        ppr, cp = self.pages_per_req, self.chunk_pages
        page_elems = c.n_kv_heads * self.page * c.head_dim
        self.block_tables, self.kv = [], []
        # host chunks are the op's leading units in chunk-major order: the oldest chunks first
        for l in range(c.n_layers):
            hu = self.attn_host_chunks[l]
            host_pages = []
            for b in range(B):
                n_chunks_b = hu // B + (1 if b < hu % B else 0)
                host_pages.append(min(ppr, n_chunks_b * cp))
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
            self.kv.append((kg, vg, kh, vh, Ph, Pg))
            self.block_tables.append(torch.from_numpy((bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda())
        # zero the host pools (finite slots beyond seq_len, dak.h) and fill prompt KV with noise
        for (kg, vg, kh, vh, Ph, Pg) in self.kv:
            n = max(Ph, 1) * page_elems
            for hp in (kh, vh):
                arr = (np.ctypeslib.as_array((__import__("ctypes").c_uint16 * n).from_address(hp[0])))
                arr[:] = 0
            kg.copy_(_bf16_rand(kg.shape, 1.0, self.gen))
            vg.copy_(_bf16_rand(vg.shape, 1.0, self.gen))
        self.positions = torch.full((B,), self.context - 1, dtype=torch.int32, device="cuda")
        self.seq_lens = self.positions + 1
        self.tokens = torch.zeros((B,), dtype=torch.int32, device="cuda")
        self.x = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.h = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.logits = torch.empty((B, c.vocab), dtype=torch.bfloat16, device="cuda")
        self.layer_args = [self._layer_args(l) for l in range(c.n_layers)]
        self.scratch = torch.empty(dak.layer_scratch_size(self.layer_args[0]), dtype=torch.uint8, device="cuda")
        for a in self.layer_args:
            a.scratch, a.scratch_bytes = self.scratch.data_ptr(), self.scratch.numel()
        # fused pre-norm: the residual stream's row statistics travel embed -> FC2 -> FC2 ... -> head
        # (one buffer: every reader of layer l's statistics finishes before FC2 of layer l rewrites it)
        self.stats = torch.zeros((1024, B, 4), dtype=torch.float32, device="cuda")
        parts = 1
        for a in self.layer_args:
            a.fuse_norm = int(self.fuse_norm)
            a.stats_in, a.stats_in_parts, a.stats_out = self.stats.data_ptr(), parts, self.stats.data_ptr()
            parts = dak.layer_stats_parts(a)
        self.head_stats_parts = parts

    def load_kv(self, K_cache, V_cache):
        """Place a given cache: K_cache[l][b] = [L_b, Hkv, d] bf16 bits (numpy) of the tokens before
        the current position, written into the tier pools named by the block table (DAK-PG)."""
        c = self.cfg
        d, Hkv, page = c.head_dim, c.n_kv_heads, self.page
        for l, (kg, vg, kh, vh, Ph, Pg) in enumerate(self.kv):
            bt = self.block_tables[l].cpu().numpy().view(np.uint32)
            pools = {}
            for name, src in (("k", K_cache[l]), ("v", V_cache[l])):
                lg = np.zeros((max(Pg, 1), Hkv, page, d), np.uint16)
                lh = np.zeros((max(Ph, 1), Hkv, page, d), np.uint16)
                for b in range(self.B):
                    arr = np.asarray(src[b])
                    for t0 in range(0, arr.shape[0], page):
                        e = int(bt[b, t0 // page])
                        pool = lh if e & 0x80000000 else lg
                        blk = arr[t0:t0 + page]
                        pool[e & 0x7FFFFFFF, :, :blk.shape[0]] = blk.transpose(1, 0, 2)
                pools[name] = (lg, lh)
            for (lg, lh), dg, dh in ((pools["k"], kg, kh), (pools["v"], vg, vh)):
                tg = torch.from_numpy(lg.view(np.int16)).cuda()
                th = torch.from_numpy(lh.view(np.int16)).cuda()
                dak.pack_kv_pages(tg, lg.shape[0] * Hkv, page, d, dg)
                dak.pack_kv_pages(th, lh.shape[0] * Hkv, page, d, dh[1])
                torch.cuda.synchronize()

    def _layer_args(self, l):
        c, L = self.cfg, self.layers[l]
        kg, vg, kh, vh, Ph, Pg = self.kv[l]
        a = dak.dak_layer_args()
        a.model, a.B, a.hidden, a.n_heads, a.n_kv_heads = dak.MODEL_OPT, self.B, c.hidden, c.n_heads, c.n_kv_heads
        a.head_dim, a.ffn, a.ln_eps = c.head_dim, c.ffn, 1e-5
        a.o, a.up, a.down = L["o"].weight(), L["up"].weight(), L["down"].weight()
        if self.fused_qkv:
            a.split_qkv = 0
            a.qkv = L["qkv"].weight()
        else:
            a.split_qkv = 1
            a.q, a.k, a.v = L["q"].weight(), L["k"].weight(), L["v"].weight()
        a.ln1_w, a.ln1_b = L["ln1_w"].data_ptr(), L["ln1_b"].data_ptr()
        a.ln2_w, a.ln2_b = L["ln2_w"].data_ptr(), L["ln2_b"].data_ptr()
        a.x = self.x.data_ptr()
        a.k_hbm, a.v_hbm = kg.data_ptr(), vg.data_ptr()
        a.k_host, a.v_host = kh[1], vh[1]
        a.block_table, a.positions, a.seq_lens = (self.block_tables[l].data_ptr(), self.positions.data_ptr(),
                                                  self.seq_lens.data_ptr())
        a.page_size, a.max_pages, a.chunk_pages = self.page, self.pages_per_req, self.chunk_pages
        a.tp_rank, a.tp_size = 0, 1
        a.cfg = dak.launch_cfg(**self.launch)
        # attention host CTAs: ~one per 8 host units (units = chunks x kv heads; one unit per warp)
        n_kvh = getattr(self, "dims", {}).get("n_kv", None) or c.n_kv_heads
        host_units = self.attn_host_chunks[l] * n_kvh
        a.attn_cfg = dak.launch_cfg(**dict(self.launch, n_cta_host=dak.attention_host_ctas(host_units)))
        # L2 warm-up chain (dak.h): the last linear of layer l warms the next layer's q (or the head)
        nxt = self.layers[l + 1]["qkv" if self.fused_qkv else "q"] if l + 1 < c.n_layers else self.head
        a.l2_prefetch_bytes = self.l2_prefetch
        if nxt.hbm is not None:
            a.next_w_hbm, a.next_w_hbm_bytes = nxt.hbm.data_ptr(), (nxt.M - nxt.h) * nxt.K * 2
        return a

    # ------------------------------------------------------------------ persistent step program
    def build_step_program(self):
        """Op table of one decode step for dak_step (embed, then per layer LN1, QKV(+KV append),
        attention[, combine], O(+residual, LN stats), LN2, FC1, FC2(+residual, LN stats), then
        LN_f and the LM head)."""
        c, B, dev = self.cfg, self.B, "cuda"
        H, F = c.hidden, c.ffn
        G = self.sms
        qkv_cols = (c.n_heads + 2 * c.n_kv_heads) * c.head_dim
        self.sp_h = torch.empty((B, H), dtype=torch.bfloat16, device=dev)
        self.sp_qkv = torch.empty((B, qkv_cols), dtype=torch.bfloat16, device=dev)
        self.sp_attn = torch.empty((B, c.n_heads * c.head_dim), dtype=torch.bfloat16, device=dev)
        self.sp_f = torch.empty((B, F), dtype=torch.bfloat16, device=dev)
        self.sp_stats = [torch.zeros((G, B, 2), dtype=torch.float32, device=dev) for _ in range(2)]
        max_chunks = self.chunks_per_req
        multi = max_chunks > 1
        n_units = B * c.n_kv_heads * max_chunks
        self.sp_part_o = torch.empty(max(1, n_units * (c.n_heads // c.n_kv_heads) * c.head_dim), dtype=torch.float32,
                                     device=dev)
        self.sp_part_lse = torch.empty(max(1, n_units * (c.n_heads // c.n_kv_heads)), dtype=torch.float32, device=dev)
        self.sp_units = []
        ops = []

        def add(**kw):
            ops.append(dak.step_op(**kw))
            return len(ops) - 1

        def lin(op: LinearOp, x, y, dep, **kw):
            return add(type=dak.STEP_LINEAR, dep=dep, w_host=op.host[1] if op.host else None, w_hbm=op.hbm, M=op.M,
                       K=op.K, h=op.h, kc=op.kc, x=x, y=y, bias=op.bias, **kw)

        prev = add(type=dak.STEP_EMBED, y=self.x, cols=H, tokens=self.tokens, positions=self.positions,
                   tok_emb=self.tok_emb, pos_emb=self.pos_emb, pos_offset=2, stats_out=self.sp_stats[0])
        for l, L in enumerate(self.layers):
            kg, vg, kh, vh, Ph, Pg = self.kv[l]
            bt = self.block_tables[l].cpu().numpy().view(np.uint32)
            uh, ug = [], []
            for b in range(B):
                for ch in range(max_chunks):
                    p0 = ch * self.chunk_pages
                    if p0 >= self.pages_per_req:
                        continue
                    (uh if bt[b, p0] & 0x80000000 else ug).append(b * max_chunks + ch)
            th = torch.tensor(uh or [0], dtype=torch.int32, device=dev)
            tg = torch.tensor(ug or [0], dtype=torch.int32, device=dev)
            self.sp_units += [th, tg]
            ln1 = add(type=dak.STEP_LAYERNORM, dep=prev, x=self.x, y=self.sp_h, cols=H, stats_in=self.sp_stats[0],
                      ln_w=L["ln1_w"], ln_b=L["ln1_b"], eps=1e-5)
            kv = dict(k_hbm=kg, v_hbm=vg, k_host=kh[1], v_host=vh[1], block_table=self.block_tables[l],
                      seq_lens=self.seq_lens, positions=self.positions, Hq=c.n_heads, Hkv=c.n_kv_heads, d=c.head_dim,
                      page_size=self.page, max_pages=self.pages_per_req, chunk_pages=self.chunk_pages)
            # q, k, v read the same LN1 output: no barrier between them; k / v epilogues append
            # the new token to the KV pools; attention depends on v (in-order completion per CTA
            # makes "every CTA finished v" imply q and k finished too)
            base = self.sp_qkv.data_ptr()
            hq = c.n_heads * c.head_dim
            hkv = c.n_kv_heads * c.head_dim
            lin(L["q"], self.sp_h, base, ln1, ldy=qkv_cols)
            lin(L["k"], self.sp_h, base + hq * 2, ln1, ldy=qkv_cols, kv_row0=0, kv_kind=1, **kv)
            qkv = lin(L["v"], self.sp_h, base + (hq + hkv) * 2, ln1, ldy=qkv_cols, kv_row0=0, kv_kind=2, **kv)
            att = add(type=dak.STEP_ATTENTION, dep=qkv, q=self.sp_qkv, q_stride=qkv_cols, out=self.sp_attn,
                      units_host=th, units_hbm=tg, n_units_host=len(uh), n_units_hbm=len(ug),
                      part_o=self.sp_part_o, part_lse=self.sp_part_lse, **kv)
            if multi:
                att = add(type=dak.STEP_COMBINE, dep=att, out=self.sp_attn, cols=B, part_o=self.sp_part_o,
                          part_lse=self.sp_part_lse, **kv)
            o = lin(L["o"], self.sp_attn, self.x, att, residual=self.x, stats_out=self.sp_stats[1])
            ln2 = add(type=dak.STEP_LAYERNORM, dep=o, x=self.x, y=self.sp_h, cols=H, stats_in=self.sp_stats[1],
                      ln_w=L["ln2_w"], ln_b=L["ln2_b"], eps=1e-5)
            f1 = lin(L["up"], self.sp_h, self.sp_f, ln2, act=dak.ACT_RELU)
            prev = lin(L["down"], self.sp_f, self.x, f1, residual=self.x, stats_out=self.sp_stats[0])
        lnf = add(type=dak.STEP_LAYERNORM, dep=prev, x=self.x, y=self.sp_h, cols=H, stats_in=self.sp_stats[0],
                  ln_w=self.lnf_w, ln_b=self.lnf_b, eps=1e-5)
        lin(self.head, self.sp_h, self.logits, lnf)
        self.step_ops = ops
        self.step_plan, self.step_buf = dak.step_compile(ops, B, cfg=self.launch)
        return self.step_plan

    # ------------------------------------------------------------------ the decode step (hot path)
    def enqueue_step(self, stream=None):
        if getattr(self, "use_step", False):
            dak.step_launch(self.step_plan, stream)
            return
        c = self.cfg
        dak.embed(self.tokens, self.positions, self.tok_emb, self.pos_emb, self.B, c.hidden, 2, self.x,
                  pdl=self.pdl, stream=stream, stats_out=self.stats if self.fuse_norm else None)
        for a in self.layer_args:
            dak.layer(a, stream)
        hw = self.head.host[1] if self.head.host else None
        if self.fuse_norm:  # LN_f fused into the LM head
            ha = dak.linear_args(hw, self.head.hbm, self.head.M, self.head.K, self.head.h, self.head.kc, self.B,
                                 self.x, self.logits, cfg=self.launch, ln_w=self.lnf_w, ln_b=self.lnf_b,
                                 ln_stats=self.stats, ln_parts=self.head_stats_parts, ln_eps=1e-5)
        else:
            dak.layernorm(self.x, self.lnf_w, self.lnf_b, self.h, self.B, c.hidden, 1e-5, pdl=self.pdl, stream=stream)
            ha = dak.linear_args(hw, self.head.hbm, self.head.M, self.head.K, self.head.h, self.head.kc, self.B,
                                 self.h, self.logits, cfg=self.launch)
        if self.B > 16:  # tcgen05 split-K partials for the head
            need = dak.linear_workspace_size(ha)
            if need:
                if getattr(self, "head_ws", None) is None or self.head_ws.numel() < need:
                    self.head_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
                ha.workspace, ha.workspace_bytes = self.head_ws.data_ptr(), self.head_ws.numel()
        dak.linear(ha, stream)

    def advance(self, stream=None):
        """Move every request to the next position (after a step appended its token's KV)."""
        if int(self.positions.max()) + 1 >= self.max_context:
            raise ValueError("decode past max_context")
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            self.positions.add_(1)
            self.seq_lens.add_(1)

    def kernels_per_step(self) -> int:
        if getattr(self, "use_step", False):
            return 1
        # [q k v | qkv] attn(+ fused KV append) [combine] o fc1 fc2
        per_layer = (5 if self.fused_qkv else 7) + (1 if self.chunks_per_req > 1 else 0)
        if self.fuse_norm:
            return 1 + per_layer * self.cfg.n_layers + 1
        return 1 + (per_layer + 2) * self.cfg.n_layers + 2

    def enable_persistent_step(self):
        if self.fused_qkv:
            raise ValueError("the persistent step program uses separate q/k/v projections: fused_qkv=False")
        self.build_step_program()
        self.use_step = True

    def capture(self, stream: torch.cuda.Stream):
        with torch.cuda.stream(stream):
            self.enqueue_step(stream)  # warm (sets function attributes outside capture)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self.enqueue_step(stream)
        self.graph = g
        return g

    def bytes_per_step(self) -> dict:
        """Algorithmic bytes read per decode step, split by tier (weights + KV)."""
        hbm = host = 0
        for op in self.linear_ops():
            hbm += (op.M - op.h) * op.K * 2
            host += op.h * op.K * 2
        c = self.cfg
        tok = 2 * c.n_kv_heads * c.head_dim * 2
        for (kg, vg, kh, vh, Ph, Pg) in self.kv:
            hp = min(Ph * self.page, self.B * self.context)
            host += tok * min(Ph * self.page, self.B * self.context)
            hbm += tok * (self.B * self.context - hp)
        return dict(hbm=hbm, host=host, total=hbm + host)

    def close(self):
        for hp in self._host_blocks:
            try:
                dak.host_free(hp)
            except Exception:
                pass
        self._host_blocks = []
