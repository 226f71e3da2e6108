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

    def as_dict(self):
        return dict(hbm_bps=self.hbm_bps, link_bps=self.link_bps,
                    host_dram_bps=self.host_dram_bps or self.link_bps, host_capacity_bytes=-1)


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
                 y_req: int = 0, unit_rows: int = 16, page_size: int = 64, chunk_pages: int = 16, seed: int = 0,
                 pdl: bool = True, congestion_control: bool = True, weights: dict | None = None,
                 host_override: dict | None = None):
        self.cfg, self.B, self.context, self.hw = cfg, batch, context, hw
        self.page, self.chunk_pages, self.unit_rows = page_size, chunk_pages, unit_rows
        self.pdl = int(pdl)
        self.launch = dict(pdl=self.pdl, congestion_control=int(congestion_control))
        self.sms = dak.device_sms()
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed)
        self._host_blocks = []
        c = cfg
        qkv_rows = (c.n_heads + 2 * c.n_kv_heads) * c.head_dim
        self.layers = []
        for i in range(c.n_layers):
            self.layers.append(dict(qkv=LinearOp(f"L{i}.qkv", qkv_rows, c.hidden),
                                    o=LinearOp(f"L{i}.o", c.hidden, c.n_heads * c.head_dim),
                                    up=LinearOp(f"L{i}.fc1", c.ffn, c.hidden),
                                    down=LinearOp(f"L{i}.fc2", c.hidden, c.ffn)))
        self.head = LinearOp("head", c.vocab, c.hidden)
        self.pages_per_req = -(-context // page_size)
        self.chunks_per_req = -(-self.pages_per_req // chunk_pages)
        self.plan = self._plan(mode, y_req, host_override)
        self._allocate(weights)
        self._kv()
        self.graph = None

    # ------------------------------------------------------------------ planning
    def linear_ops(self):
        for L in self.layers:
            yield from (L["qkv"], L["o"], L["up"], L["down"])
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
            op.kc = dak.default_kc(op.M - op.h, op.K, self.sms - 1)
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
        for i, L in enumerate(self.layers):
            for key, op in L.items():
                W = weights[f"L{i}.{key}"] if weights else None
                self._fill_linear(op, W)
                op.bias = weights[f"L{i}.{key}.b"] if weights else _bf16_rand((op.M,), 0.02, self.gen)
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
        a.qkv, a.o, a.up, a.down = L["qkv"].weight(), L["o"].weight(), L["up"].weight(), L["down"].weight()
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
        a.attn_cfg = dak.launch_cfg(**self.launch)
        return a

    # ------------------------------------------------------------------ the decode step (hot path)
    def enqueue_step(self, stream=None):
        c = self.cfg
        dak.embed(self.tokens, self.positions, self.tok_emb, self.pos_emb, self.B, c.hidden, 2, self.x,
                  pdl=self.pdl, stream=stream)
        for a in self.layer_args:
            dak.layer(a, stream)
        dak.layernorm(self.x, self.lnf_w, self.lnf_b, self.h, self.B, c.hidden, 1e-5, pdl=self.pdl, stream=stream)
        ha = dak.linear_args(self.head.host[1] if self.head.host else None, self.head.hbm, self.head.M, self.head.K,
                             self.head.h, self.head.kc, self.B, self.h, self.logits, cfg=self.launch)
        dak.linear(ha, stream)

    def kernels_per_step(self) -> int:
        return 1 + 9 * self.cfg.n_layers + 2

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
