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

from dataclasses import dataclass

import torch

from . import dak, tp
from .engine import HW, _DecodeEngine, _bf16_rand


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


class DakLlama(_DecodeEngine):
    """Decode step of one tensor-parallel rank over HBM + pinned host memory at planned ratios."""

    family = dak.MODEL_LLAMA

    def __init__(self, cfg: LlamaConfig, batch: int, context: int, hw: HW, tp_rank: int = 0, tp_size: int = 1,
                 comm=None, mode: int = dak.PLAN_BALANCED, y_req: int = 0, unit_rows: int = 16, page_size: int = 64,
                 chunk_pages: int = 0, seed: int = 0, pdl: bool = True, congestion_control: bool = True,
                 weights: dict | None = None, n_cta_host: int = 2, fuse_norm: bool | None = None,
                 nvls: bool = False, host_inflight_kb: int = 0):
        self.cfg = cfg
        self.rank, self.world, self.comm = tp_rank, tp_size, comm
        # operand transforms fused into the linears only at small batch: above 16 columns every CTA
        # would re-normalise / re-activate the whole operand (measured 3-8x slower than one kernel)
        self.fuse_norm = (batch <= 16) if fuse_norm is None else bool(fuse_norm)
        self.dims = tp.local_dims(cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.vocab, tp_size)
        self.n_kv_local, self.head_dim = self.dims["n_kv"], cfg.head_dim
        self._init_common(batch, context, hw, unit_rows, page_size, chunk_pages, None, self.dims["n_kv"], pdl,
                          congestion_control, n_cta_host, seed + 7919 * tp_rank, host_inflight_kb=host_inflight_kb)
        self._plan(mode, y_req)
        self._allocate(weights)
        self._kv_pools(self.dims["n_kv"], cfg.head_dim)
        # NVLS combine (unfused TP path): o / down partials into a symmetric NCCL window, one
        # combine kernel with the reduction in the NVSwitch (dak_nvls_create; collective call)
        self.nvls = None
        if nvls and comm and not self.fuse_norm:
            self.nvls, _ = dak.nvls_create(comm, batch * cfg.hidden * 2, batch)
        self._layer_setup()

    def _model_desc(self):
        c = self.cfg
        return dak.model(dak.MODEL_LLAMA, c.n_layers, c.hidden, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab,
                         tp_size=self.world, fused_qkv=1, fused_gate_up=1, include_head=1)

    def _allocate(self, weights):
        """weights: FULL logical parameters as device bf16 tensors (names as oracle/layer.py), sharded
        here for this rank; None -> random weights of the shard's shapes."""
        c, dev = self.cfg, "cuda"
        loc = None
        if weights:
            loc = tp.shard_llama(weights, self.rank, self.world, c.n_heads, c.n_kv_heads, c.head_dim)
        for i, L in enumerate(self.layers):
            for key, op in list(L.items()):
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

    def _layer_setup(self):
        c, B = self.cfg, self.B
        self.x = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.hnorm = torch.empty((B, c.hidden), dtype=torch.bfloat16, device="cuda")
        self.logits = torch.empty((B, self.dims["vocab"]), dtype=torch.bfloat16, device="cuda")
        self.layer_args = [self._layer_args(l) for l in range(c.n_layers)]
        self.scratch = torch.zeros(dak.layer_scratch_size(self.layer_args[0]), dtype=torch.uint8, device="cuda")
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
        self._load_kv(K_cache, V_cache, self.dims["n_kv"], self.cfg.head_dim)

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
        a.nvls = self.nvls
        a.cfg = dak.launch_cfg(**self.launch)
        a.attn_cfg = dak.launch_cfg(**self.attn_launch)
        return a

    # ------------------------------------------------------------------ the decode step (hot path)
    def enqueue_step(self, stream=None):
        c = self.cfg
        dak.embed(self.tokens, None, self.tok_emb, None, self.B, c.hidden, 0, self.x, pdl=self.pdl, stream=stream,
                  stats_out=self.stats if self.fuse_norm else None)
        for a in self.layer_args:
            dak.layer(a, stream)
        if self.fuse_norm:  # final RMSNorm fused into the LM head
            ha = self._head_args(self.x, self.logits, ln_w=self.lnf_w, ln_stats=self.stats,
                                 ln_parts=self.head_stats_parts, ln_rms=1, ln_eps=c.rms_eps)
        else:
            dak.rmsnorm(self.x, self.lnf_w, self.hnorm, self.B, c.hidden, c.rms_eps, pdl=self.pdl, stream=stream)
            ha = self._head_args(self.hnorm, self.logits)
        dak.linear(ha, stream)

    def close(self):
        if getattr(self, "nvls", None):
            dak.nvls_destroy(self.nvls)
            self.nvls = None
        super().close()

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
