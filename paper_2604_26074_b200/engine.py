"""DAK decode engines, built on the C ABI (PAPER §4).

Setup (once, per GPU): the op list of one decode step (dak_decode_ops: C_i, units, FLOPs, T_i;
P:L383-388) -> dak_plan_ratios (greedy per-op ratios) -> byte placement (linear: host =
the leading rows; attention: dak_kv_place, the oldest split-KV chunks) -> DAK-KC / DAK-PG
packing into HBM and pinned mapped host memory -> one decode step captured in a CUDA graph.
Step (hot path): embed -> layers (dak_layer) -> final norm + LM head, every weight and KV page
streamed by the library's split-source kernels.

This module holds only setup and marshalling: every number of the method (op profile, ratios,
placement, CTA roles) comes from the library. torch is used for device memory, streams and graphs
only. This module never imports the CPU oracle.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

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
    host_capacity_bytes: int = -1

    @classmethod
    def from_calibration(cls, cal: dict, peak_flops: float = 1.3554e15):
        """The planner's machine model measured by dak_calibrate: B_g and B_h at the
        chosen congestion-control point (concurrent rates), tau = the link latency."""
        return cls(hbm_bps=cal["hbm_bps"], link_bps=cal["link_bps"], peak_flops=peak_flops,
                   host_latency_s=cal["host_latency_s"])

    def as_dict(self):
        return dict(hbm_bps=self.hbm_bps, link_bps=self.link_bps,
                    host_dram_bps=self.host_dram_bps or self.link_bps, host_capacity_bytes=self.host_capacity_bytes,
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


class _DecodeEngine:
    """Shared setup of one GPU's decode step: planning, placement, KV pools, graph capture."""

    family = dak.MODEL_OPT
    # op-list role -> key of the layer dict holding the LinearOp
    ROLE_KEY = dict(qkv="qkv", q="q", k="k", v="v", o="o", up="up", gate_up="up", down="down")

    def _init_common(self, batch, context, hw, unit_rows, page_size, chunk_pages, max_context, n_kv_local,
                     pdl, congestion_control, n_cta_host, seed, evict_first=True, kv_replan=False,
                     host_inflight_kb=0):
        self.B, self.context, self.hw = batch, context, hw
        self.cur_len = context  # tokens every request holds for the next step (host mirror of seq_lens)
        # KV placement across decode steps (reading R23): pools sized for any placement, re-placed as
        # the requests grow (advance -> replan)
        self.kv_replan = bool(kv_replan)
        self.page, self.unit_rows = page_size, unit_rows
        self.max_context = max(context, max_context or context)
        self.pages_per_req = -(-self.max_context // page_size)
        if not chunk_pages:  # split-KV chunk: about one (request, kv head, chunk) unit per two warp slots (measured best)
            units_1 = batch * n_kv_local * self.pages_per_req
            chunk_pages = max(1, min(16, units_1 // (148 * 4)))
        self.chunk_pages = chunk_pages
        self.chunks_per_req = -(-self.pages_per_req // chunk_pages)
        self.pdl = int(pdl)
        self.n_cta_host = n_cta_host
        # congestion control: host CTAs and host bytes in flight (dak_calibrate's choice when given;
        # 0 = the library's defaults)
        self.launch = dict(pdl=self.pdl, congestion_control=int(congestion_control), n_cta_host=n_cta_host,
                           l2_policy=0 if evict_first else 1, host_inflight_kb=int(host_inflight_kb))
        # attention: host CTAs chosen by the library from the block table (dak_attention auto mode)
        self.attn_launch = dict(self.launch, n_cta_host=0)
        self.sms = dak.device_sms()
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed)
        self._host_blocks = []
        self.graph = None

    # ------------------------------------------------------------------ planning
    def _model_desc(self) -> dak.dak_model:
        raise NotImplementedError

    def _plan(self, mode, y_req, host_override=None):
        """dak_decode_ops -> dak_plan_ratios; builds self.layers / self.head from the op list."""
        self.model_desc = self._model_desc()
        ops = dak.decode_ops(self.model_desc, self.B, self.context, self.unit_rows, self.chunk_pages * self.page,
                             self.hw.peak_flops, self.hw.peak_flops)
        self.plan_ops = ops
        plan, self.objective = dak.plan_ratios(self.hw.as_dict(), ops, y_req, mode)
        self.plan = plan
        n_layers = max(o["layer"] for o in ops) + 1
        self.layers = [dict() for _ in range(n_layers)]
        self.attn_host_chunks = [0] * n_layers
        self.head = None
        self.attn_units = [0] * n_layers
        for o, p in zip(ops, plan):
            if o["role"] == "attn":
                self.attn_host_chunks[o["layer"]] = p["host_units"]
                self.attn_units[o["layer"]] = o["n_units"]
                continue
            name = "head" if o["role"] == "head" else f"L{o['layer']}.{o['role']}"
            op = LinearOp(name, o["M"], o["K"])
            op.h = min(op.M, p["host_units"] * self.unit_rows)
            if host_override and o["role"] in host_override:
                op.h = host_override[o["role"]]
            if o["role"] == "head":
                self.head = op
            else:
                self.layers[o["layer"]][self.ROLE_KEY[o["role"]]] = op
            # KC = 64 where the tcgen05 path runs (its canonical SWIZZLE_128B operands): above 16
            # batch columns, and at 9..16 for ops with >= 128 rows per SM (dak_linear picks tcgen05
            # there); else the widest KC whose stage holds the CTA's rows (dak_linear_choose_kc)
            n_host = min(self.n_cta_host, op.h) if op.h > 0 else 0
            rows = max(-(-op.h // max(n_host, 1)) if op.h else 0, -(-(op.M - op.h) // (self.sms - n_host)))
            tc = self.B > 16 or (self.B > 8 and op.M >= 128 * self.sms)
            op.kc = 64 if tc else dak.choose_kc(rows, op.K)
        return plan

    def linear_ops(self):
        for L in self.layers:
            for key in ("qkv", "q", "k", "v", "o", "up", "down"):
                if isinstance(L.get(key), LinearOp):
                    yield L[key]
        yield self.head

    # ------------------------------------------------------------------ placement + packing
    def _alloc_host(self, nbytes):
        hp, dp = dak.host_alloc(max(nbytes, 16), numa_node=self.numa_node)
        self._host_blocks.append(hp)
        return hp, dp

    @property
    def numa_node(self) -> int:
        if not hasattr(self, "_numa"):
            self._numa = dak.device_numa_node()
        return self._numa

    def _fill_linear(self, op: LinearOp, W):
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

    def _kv_pools(self, n_kv_local, head_dim):
        """Per layer: dak_kv_place's block table (oldest chunks on the host, chunk-major), the two
        tier pools (prompt KV drawn N(0, 1) in HBM, host pools zeroed then packed by load_kv)."""
        B, ppr = self.B, self.pages_per_req
        page_elems = n_kv_local * self.page * head_dim
        self.block_tables, self.kv, self.kv_host_tokens, self.block_tables_np = [], [], [], []
        for l in range(len(self.layers)):
            bt, Ph, Pg, ht = dak.kv_place([self.context] * B, self.page, ppr, self.chunk_pages,
                                          self.attn_host_chunks[l])
            self.block_tables_np.append(bt)
            if self.kv_replan:  # room for every page in either pool (placements change as requests grow)
                Ph, Pg = B * ppr, B * ppr
            kg = torch.zeros(max(Pg, 1) * page_elems, dtype=torch.bfloat16, device="cuda")
            vg = torch.zeros_like(kg)
            kh = self._alloc_host(max(Ph, 1) * page_elems * 2)
            vh = self._alloc_host(max(Ph, 1) * page_elems * 2)
            for hp in (kh, vh):  # finite slots beyond seq_len (dak.h)
                ctypes.memset(hp[0], 0, max(Ph, 1) * page_elems * 2)
            kg.copy_(_bf16_rand(kg.shape, 1.0, self.gen))
            vg.copy_(_bf16_rand(vg.shape, 1.0, self.gen))
            self.kv.append((kg, vg, kh, vh, Ph, Pg))
            self.kv_host_tokens.append(ht)
            self.block_tables.append(torch.from_numpy(bt).cuda())
        self.positions = torch.full((B,), self.context - 1, dtype=torch.int32, device="cuda")
        self.seq_lens = self.positions + 1
        self.tokens = torch.zeros((B,), dtype=torch.int32, device="cuda")

    def _load_kv(self, K_cache, V_cache, n_kv_local, d):
        """K_cache[l][b] = [L_b, Hkv, d] bf16 bits (numpy) of the cached tokens, written into the tier
        pools the block table names (DAK-PG)."""
        page = self.page
        for l, (kg, vg, kh, vh, Ph, Pg) in enumerate(self.kv):
            bt = self.block_tables[l].cpu().numpy().view(np.uint32)
            pools = {}
            for name, src in (("k", K_cache[l]), ("v", V_cache[l])):
                lg = np.zeros((max(Pg, 1), n_kv_local, page, d), np.uint16)
                lh = np.zeros((max(Ph, 1), n_kv_local, page, d), np.uint16)
                for b in range(self.B):
                    arr = np.asarray(src[b])
                    for t0 in range(0, arr.shape[0], page):
                        e = int(bt[b, t0 // page])
                        pool = lh if e & dak.HOST_BIT else lg
                        blk = arr[t0:t0 + page]
                        pool[e & 0x7FFFFFFF, :, :blk.shape[0]] = blk.transpose(1, 0, 2)
                pools[name] = (lg, lh)
            for (lg, lh), dg, dh in ((pools["k"], kg, kh), (pools["v"], vg, vh)):
                dak.pack_kv_pages(torch.from_numpy(lg.view(np.int16)).cuda(), lg.shape[0] * n_kv_local, page, d, dg)
                dak.pack_kv_pages(torch.from_numpy(lh.view(np.int16)).cuda(), lh.shape[0] * n_kv_local, page, d, dh[1])
                torch.cuda.synchronize()

    def _head_args(self, x, out, **kw):
        hw = self.head.host[1] if self.head.host else None
        ha = dak.linear_args(hw, self.head.hbm, self.head.M, self.head.K, self.head.h, self.head.kc, self.B, x, out,
                             cfg=self.launch, **kw)
        if self.B > 16:  # tcgen05 split-K partials for the head
            need = dak.linear_workspace_size(ha)
            if need:
                if getattr(self, "head_ws", None) is None or self.head_ws.numel() < need:
                    self.head_ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
                ha.workspace, ha.workspace_bytes = self.head_ws.data_ptr(), self.head_ws.numel()
        return ha

    # ------------------------------------------------------------------ step
    def advance(self, stream=None):
        """Move every request to the next position (after a step appended its token's KV). With
        kv_replan, a step that opens a new split-KV chunk first re-places the KV (replan)."""
        if int(self.positions.max()) + 1 >= self.max_context:
            raise ValueError("decode past max_context")
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            self.positions.add_(1)
            self.seq_lens.add_(1)
        self.cur_len += 1
        if self.kv_replan and (self.cur_len - 1) % (self.chunk_pages * self.page) == 0:
            self.replan(stream)

    def replan(self, stream=None):
        """KV placement across decode steps (reading R23 of DESIGN.md): every
        attention op keeps the host ratio the planner gave it, x = host units / units at planning
        (per-op ratio x_i), as its chunk count grows: host units = round-half-up(x * units),
        the R6 rounding. dak_kv_replace gives the new block table (chunk-major oldest chunks on the
        host, pages keep their slot unless their tier changes) and the page moves, dak_kv_migrate
        copies the moved pages on the device, then the table the captured graph reads is rewritten
        in place (stream-ordered before the next replay)."""
        if not self.kv_replan:
            raise ValueError("replan needs kv_replan=True (pools sized for any placement)")
        B, ppr, cp, page = self.B, self.pages_per_req, self.chunk_pages, self.page
        L = self.cur_len
        n_new = B * (-(-(-(-L // page)) // cp))
        s = stream or torch.cuda.current_stream()
        keep = []
        with torch.cuda.stream(s):
            for l, (kg, vg, kh, vh, Ph, Pg) in enumerate(self.kv):
                h0, n0 = self.attn_host_chunks[l], self.attn_units[l]
                hu = min(n_new, (2 * h0 * n_new + n0) // (2 * n0)) if n0 else 0
                new, moves = dak.kv_replace(self.block_tables_np[l], [L] * B, page, ppr, cp, hu, Ph, Pg)
                if len(moves):
                    mv = torch.from_numpy(moves).cuda()
                    keep.append(mv)
                    dak.kv_migrate(mv, len(moves), self.n_kv_local, page, self.head_dim, kg, vg, kh[1], vh[1], s)
                self.block_tables[l].copy_(torch.from_numpy(new))
                self.block_tables_np[l] = new
                hp = ((new.view(np.uint32) & dak.HOST_BIT) != 0).sum(axis=1)
                self.kv_host_tokens[l] = int(np.minimum(hp * page, L).sum())
        s.synchronize()

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
        """Algorithmic bytes read per decode step, split by tier (weights + KV of the context)."""
        hbm = host = 0
        for op in self.linear_ops():
            hbm += (op.M - op.h) * op.K * 2
            host += op.h * op.K * 2
        tok = 2 * self.n_kv_local * self.head_dim * 2
        for ht in self.kv_host_tokens:
            host += tok * ht
            hbm += tok * (self.B * self.cur_len - ht)
        return dict(hbm=hbm, host=host, total=hbm + host)

    def close(self):
        for hp in self._host_blocks:
            try:
                dak.host_free(hp)
            except Exception:
                pass
        self._host_blocks = []


class DakOPT(_DecodeEngine):
    """OPT decode step over HBM + pinned host memory at per-op planned ratios."""

    family = dak.MODEL_OPT

    def __init__(self, cfg: OPTConfig, batch: int, context: int, hw: HW, mode: int = dak.PLAN_BALANCED,
                 y_req: int = 0, unit_rows: int = 16, page_size: int = 64, chunk_pages: int = 0, seed: int = 0,
                 pdl: bool = True, congestion_control: bool = True, weights: dict | None = None,
                 host_override: dict | None = None, n_cta_host: int = 2, l2_prefetch: int = 0,
                 evict_first: bool = True, fuse_norm: bool = True, fused_qkv: bool = True,
                 max_context: int | None = None, kv_replan: bool = False, host_inflight_kb: int = 0):
        self.cfg = cfg
        self.n_kv_local, self.head_dim = cfg.n_kv_heads, cfg.head_dim
        self._init_common(batch, context, hw, unit_rows, page_size, chunk_pages, max_context, cfg.n_kv_heads,
                          pdl, congestion_control, n_cta_host, seed, evict_first, kv_replan, host_inflight_kb)
        self.l2_prefetch = int(l2_prefetch)
        self.fuse_norm = bool(fuse_norm)
        # one [q; k; v] projection per layer (one launch reading x once; reading R18); the paper's
        # op list has the three projections separately
        self.fused_qkv = bool(fused_qkv)
        self._plan(mode, y_req, host_override)
        self._allocate(weights)
        self._kv_pools(cfg.n_kv_heads, cfg.head_dim)
        self._layer_setup()

    def _model_desc(self):
        c = self.cfg
        return dak.model(dak.MODEL_OPT, c.n_layers, c.hidden, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab,
                         tp_size=1, fused_qkv=int(self.fused_qkv), fused_gate_up=0, include_head=1)

    def kv_bytes_per_layer(self) -> int:
        c = self.cfg
        return 2 * c.n_kv_heads * c.head_dim * 2 * self.B * self.context

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

    def _layer_setup(self):
        c, B = self.cfg, self.B
        self.x = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.h = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.logits = torch.empty((B, c.vocab), dtype=torch.bfloat16, device="cuda")
        self.layer_args = [self._layer_args(l) for l in range(c.n_layers)]
        self.scratch = torch.zeros(dak.layer_scratch_size(self.layer_args[0]), dtype=torch.uint8, device="cuda")
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
        self._load_kv(K_cache, V_cache, self.cfg.n_kv_heads, self.cfg.head_dim)

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
        a.attn_cfg = dak.launch_cfg(**self.attn_launch)
        # L2 warm-up chain (dak.h): the last linear of layer l warms the next layer's q (or the head)
        nxt = self.layers[l + 1]["qkv" if self.fused_qkv else "q"] if l + 1 < c.n_layers else self.head
        a.l2_prefetch_bytes = self.l2_prefetch
        if nxt.hbm is not None:
            a.next_w_hbm, a.next_w_hbm_bytes = nxt.hbm.data_ptr(), (nxt.M - nxt.h) * nxt.K * 2
        return a

    # ------------------------------------------------------------------ the decode step (hot path)
    def enqueue_step(self, stream=None):
        c = self.cfg
        dak.embed(self.tokens, self.positions, self.tok_emb, self.pos_emb, self.B, c.hidden, 2, self.x,
                  pdl=self.pdl, stream=stream, stats_out=self.stats if self.fuse_norm else None)
        for a in self.layer_args:
            dak.layer(a, stream)
        if self.fuse_norm:  # LN_f fused into the LM head
            ha = self._head_args(self.x, self.logits, ln_w=self.lnf_w, ln_b=self.lnf_b, ln_stats=self.stats,
                                 ln_parts=self.head_stats_parts, ln_eps=1e-5)
        else:
            dak.layernorm(self.x, self.lnf_w, self.lnf_b, self.h, self.B, c.hidden, 1e-5, pdl=self.pdl, stream=stream)
            ha = self._head_args(self.h, self.logits)
        dak.linear(ha, stream)

    def kernels_per_step(self) -> int:
        # [q k v | qkv] attn(+ fused KV append) [combine] o fc1 fc2
        per_layer = (5 if self.fused_qkv else 7) + (1 if self.chunks_per_req > 1 else 0)
        if self.fuse_norm:
            return 1 + per_layer * self.cfg.n_layers + 1
        return 1 + (per_layer + 2) * self.cfg.n_layers + 2
