/*
 * dak.h — C ABI of the B200-native DAK decode hot path (arxiv 2604.26074, "DAK: Direct-Access-
 * Enabled GPU Memory Offloading with Optimal Efficiency for LLM Inference").
 *
 * Citations: P:L<n> = /root/reference/PAPER.md line n (section noted), S:L<n> = SPEC.md line n.
 *
 * Conventions (all entry points):
 *  - Every call returns dak_status (DAK_OK == 0). No exception crosses the ABI. On failure
 *    dak_last_error() returns a thread-local, human-readable message (valid until the next call
 *    on the same thread).
 *  - The CALLER owns every buffer. Op calls never allocate device or host memory; workspace is
 *    passed in and its size comes from the pure *_workspace_size queries. dak_host_alloc /
 *    dak_host_free are separate setup helpers for the host tier.
 *  - Device pointers must be 16-byte aligned (bulk-copy requirement) or the call returns
 *    DAK_EINVAL. Host-tier pointers must be pinned AND mapped into the device address space
 *    (cudaHostAlloc(cudaHostAllocMapped|cudaHostAllocPortable), cudaHostRegister(...Mapped) or
 *    dak_host_alloc); with UVA the host pointer is the device pointer.
 *  - Op calls are asynchronous on the given stream (a cudaStream_t passed as void*; NULL = the
 *    legacy default stream). Asynchronous CUDA errors surface at the caller's next sync.
 *    Op calls contain no host synchronisation and no allocation, so they can be captured in a
 *    CUDA graph. Calls on distinct streams are thread-safe.
 *  - bf16 tensors are IEEE bfloat16 bit patterns (uint16). Accumulation is fp32; outputs are
 *    rounded to bf16 with round-to-nearest-even.
 */
#ifndef DAK_H_
#define DAK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dak_status;
#define DAK_OK 0
#define DAK_EINVAL 1        /* bad argument (shape, alignment, mode, NULL)                 */
#define DAK_ECAPACITY 2     /* required host bytes exceed offloadable bytes / host capacity */
#define DAK_EUNSUPPORTED 3  /* valid request outside what this build implements            */
#define DAK_ECUDA 4         /* a CUDA runtime/driver call failed (message has the detail)  */
#define DAK_ENCCL 5         /* an NCCL call failed                                          */

typedef void* dak_stream_t; /* cudaStream_t */

const char* dak_last_error(void);
const char* dak_version(void);
/* Number of SMs of the current device (launch sizing; DAK_ECUDA without a device). */
dak_status dak_device_sms(int32_t* sms);

/* Launch-timeline tracing (debug/measurement; not thread-safe). While enabled, each of the next
 * max_launches per-op launches (linear, attention, combine, KV append, LayerNorm, embed) records
 * globaltimer stamps (ns) into dev_buf[launch][cta < 1024][4]: 0 CTA start, 1 dependency wait
 * returned, 2 first pipeline stage consumed, 3 CTA done (0 where a kernel has no such point).
 * dev_buf: device, >= max_launches * 32 KB, zeroed by the caller. NULL disables. Launches
 * recorded under CUDA-graph capture stamp on every replay. */
dak_status dak_trace_enable(void* dev_buf, int32_t max_launches);
int32_t dak_trace_count(void);
/* kind: 1 linear (a = M, b = K), 2 attention, 3 combine, 4 KV append, 5 LayerNorm, 6 embed,
 * 7 split-K reduce (a = M, b = splits), 8 prefill attention (a = B, b = T), 9 residual + RMSNorm
 * (a = rows, b = cols), 10 silu * up (a = rows, b = F). */
dak_status dak_trace_launch(int32_t i, int32_t* kind, int64_t* a, int64_t* b, int32_t* grid);

/* =============================================================================================
 * 1. Planner — greedy per-op offload ratios (§3.2; App. A)
 * ============================================================================================= */

/* Machine model. B_g = hbm_bps; B_h = min(link_bps, host_dram_bps) (P:L216 footnote).
 * Bandwidths in bytes/s (> 0). host_capacity_bytes < 0 means unlimited. host_latency_s >= 0
 * (latency-aware extension): an op reading any host byte pays it once,
 * T_h = y/B_h + tau, which moves each op's balance point to T* = max(T, (C + B_h tau)/(B_g + B_h));
 * 0 reproduces the paper's model exactly. */
typedef struct {
  double hbm_bps;
  double link_bps;
  double host_dram_bps;
  int64_t host_capacity_bytes;
  double host_latency_s;
} dak_hw;

#define DAK_OP_LINEAR 0     /* C_i = weight bytes                              (P:L422 fn) */
#define DAK_OP_ATTENTION 1  /* C_i = KV-cache bytes                            (P:L422 fn) */

/* One offloadable operation. The op's matrix is cut into n_units placement units (linear:
 * unit_rows output rows; attention: split-KV chunks or whole requests); host units are
 * the LEADING units. total_bytes = C_i; every unit is unit_bytes except possibly the
 * last: (n_units-1)*unit_bytes < total_bytes <= n_units*unit_bytes. t_comp_s = T_comp (>= 0). */
typedef struct {
  int32_t kind;
  int32_t reserved;
  int64_t n_units;
  int64_t unit_bytes;
  int64_t total_bytes;
  double t_comp_s;
} dak_op;

typedef struct {
  int64_t host_units;  /* units placed in host memory (leading units)                      */
  int64_t host_bytes;  /* = host_units*unit_bytes, or total_bytes when all units are host    */
  double ratio;        /* host_units / n_units (x_i of P:L466)                               */
  int32_t phase;       /* last greedy phase that gave this op budget: 0 none, 1..3 */
  int32_t reserved;
  double latency_s;    /* max(T_comp, (C-y)/B_g, y/B_h) at the planned y   */
} dak_op_plan;

#define DAK_PLAN_EXACT 0    /* place >= y_req_bytes on host, greedy phases 1->3 (R4)  */
#define DAK_PLAN_BALANCED 1 /* place max(y_req, sum of memory-bound turning points)  */

/* Three-phase greedy at unit granularity; readings R1, R4-R6 of DESIGN.md.
 * Deterministic and bit-identical to oracle/planner.py:plan_units (IEEE double, fixed formula
 * order, no FMA contraction). out: caller array of n_ops. objective_s (nullable): sum of the
 * per-op latencies (App. A objective).
 * Errors: DAK_EINVAL (n_ops <= 0, NULL, non-positive bandwidth, inconsistent units, y_req < 0,
 * bad mode); DAK_ECAPACITY (y_req > sum total_bytes or > host capacity). */
dak_status dak_plan_ratios(const dak_hw* hw, const dak_op* ops, int32_t n_ops, int64_t y_req_bytes,
                           int32_t mode, dak_op_plan* out, double* objective_s);

/* =============================================================================================
 * 1b. Planner inputs and placement. Pure host functions.
 * ============================================================================================= */

/* a1 -- capacity -> global host budget (§3.2: "the offload ratio is decided by the memory
 * footprint and the GPU capacity"; Fig. 8). footprint = weight_bytes + kv_bytes;
 * *y_req_bytes = max(0, footprint - hbm_budget_bytes) (the bytes that must live on the host);
 * *ratio (nullable) = y_req / footprint (R of P:L880), 0 for an empty footprint.
 * Errors: DAK_EINVAL (NULL output, negative size); DAK_ECAPACITY (host_capacity_bytes >= 0 and the
 * overflow exceeds it). host_capacity_bytes < 0: unlimited. */
dak_status dak_global_offload_bytes(int64_t weight_bytes, int64_t kv_bytes, int64_t hbm_budget_bytes,
                                    int64_t host_capacity_bytes, int64_t* y_req_bytes, double* ratio);

#define DAK_MODEL_OPT 0   /* pre-LayerNorm, biases, ReLU MLP (OPT family)            */
#define DAK_MODEL_LLAMA 1 /* pre-RMSNorm, no biases, rotary, GQA, SwiGLU MLP (BASELINE C3)   */

/* Decoder-only transformer shape. With tp_size > 1 the op list is ONE rank's Megatron shard:
 * q / k / v / gate / up / LM head split by output rows, o / down by input columns (heads, kv heads,
 * ffn and vocab must divide by tp_size). */
typedef struct {
  int32_t family;        /* DAK_MODEL_OPT | DAK_MODEL_LLAMA                                       */
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
  int32_t tp_size;       /* 0 / 1: unsharded                                                      */
  int32_t fused_qkv;     /* 1: one [q; k; v] op per layer (reading R18); 0: q, k, v (P:L981 fn)   */
  int32_t fused_gate_up; /* Llama: 1: one [gate; up] op of 2 ffn rows; 0: gate, up                */
  int32_t include_head;  /* 1: the LM head as the last op (OPT: the tied token embedding)         */
} dak_model;

#define DAK_ROLE_Q 0
#define DAK_ROLE_K 1
#define DAK_ROLE_V 2
#define DAK_ROLE_QKV 3
#define DAK_ROLE_O 4
#define DAK_ROLE_UP 5        /* OPT fc1; Llama up                                                 */
#define DAK_ROLE_DOWN 6      /* OPT fc2; Llama down                                               */
#define DAK_ROLE_GATE 7
#define DAK_ROLE_GATE_UP 8
#define DAK_ROLE_ATTENTION 9
#define DAK_ROLE_HEAD 10

typedef struct {
  int32_t layer;  /* -1: the LM head                                                             */
  int32_t role;   /* DAK_ROLE_*                                                                   */
  int64_t M, K;   /* linear: output rows, input columns of this shard; attention: B*context, d   */
  double flops;   /* 2*B*M*K (linear); 4*B*context*(Hq d) (decode attention)     */
} dak_op_desc;

/* a2 -- the per-op profile of one decode step (§3.2, P:L422 footnote "C_i is the
 * weight or KV size", P:L981 footnote "offloadable ops are the linear layers and attention";
 * S:L135-143). Order: for each layer its linear ops in model order ([q k v | qkv], o, OPT: fc1 fc2 /
 * Llama: [gate up | gate_up], down) then its attention op; the LM head last.
 * Linear op: C = 2 M K bytes, units of unit_rows output rows (n = ceil(M / unit_rows), unit_bytes =
 * 2 unit_rows K; reading R8), T = flops / peak_flops_linear.
 * Attention op (the new token of each of `batch` requests over `context` cached tokens, this shard's
 * kv heads): C = 2 (K, V) * Hkv d * 2 B * batch * context; units = split-KV chunks of chunk_tokens
 * tokens of one request (all its kv heads): n = batch * ceil(context / chunk_tokens), unit_bytes =
 * ceil(C / n) (reading R15); T = flops / peak_flops_attn.
 * T values are IEEE double with the written operation order (bit-identical to the oracle).
 * ops / desc (each nullable; both NULL = count query): caller arrays of `capacity` entries.
 * *n_ops = number of ops. Errors: DAK_EINVAL (NULL model / n_ops, non-positive size or peak,
 * n_heads % n_kv_heads, dims not divisible by tp_size, capacity too small). */
dak_status dak_decode_ops(const dak_model* model, int32_t batch, int64_t context, int32_t unit_rows,
                          int32_t chunk_tokens, double peak_flops_linear, double peak_flops_attn, dak_op* ops,
                          dak_op_desc* desc, int32_t capacity, int32_t* n_ops);

/* a4 (attention) -- KV placement of one layer ("tile row 0 resides in host memory",
 * P:L631 KV partitioned for SplitK_FlashAttn; readings R7, R15 of DESIGN.md). Request b holds
 * seq_lens[b] tokens in ceil(seq_lens[b] / page_size) filled pages; its block-table row has
 * max_pages entries (pages past the filled ones take later decode tokens, in HBM). The op's
 * host_units (planner units: split-KV chunks of chunk_pages pages) are the OLDEST chunks, taken
 * chunk-major: chunk 0 of requests 0..B-1, then chunk 1, ... (chunks that exist only). Host pages
 * get host-pool indices 0, 1, ... in (request, page) order, all other entries HBM-pool indices
 * likewise; a host entry is index | 0x80000000 (dak_attention's tier bit).
 * block_table: caller host array [B * max_pages] (int32). n_host_pages / n_hbm_pages (nullable):
 * pool sizes in pages; host_tokens (nullable): tokens whose K/V rows live on the host.
 * Errors: DAK_EINVAL (bad sizes, seq_len beyond max_pages pages, host_units > existing chunks). */
dak_status dak_kv_place(int32_t B, const int32_t* seq_lens, int32_t page_size, int32_t max_pages, int32_t chunk_pages,
                        int64_t host_units, int32_t* block_table, int32_t* n_host_pages, int32_t* n_hbm_pages,
                        int64_t* host_tokens);

/* a4 across decode steps (reading R23): the requests grew to
 * seq_lens and the planner gave the op host_units; every block-table entry takes the tier of
 * dak_kv_place's chunk-major placement for these lengths and units. An entry keeps its pool slot when
 * its tier is unchanged; an entry whose tier changes takes the lowest slot of the destination pool
 * (host_pool_pages / hbm_pool_pages pages) that old_table does not reference -- so slots freed here
 * are reused only by a later call, and every copy reads a slot nothing writes. Outputs: new_table
 * [B * max_pages] (caller host array, != old_table) and moves [n_moves][2] (old entry, new entry)
 * in (request, page) order, for dak_kv_migrate. Pure host computation.
 * Errors: DAK_EINVAL (bad sizes, old slot outside its pool, more than max_moves moves),
 * DAK_ECAPACITY (a destination pool has no free slot). */
dak_status dak_kv_replace(int32_t B, const int32_t* seq_lens, int32_t page_size, int32_t max_pages, int32_t chunk_pages,
                          int64_t host_units, int32_t host_pool_pages, int32_t hbm_pool_pages, const int32_t* old_table,
                          int32_t* new_table, int32_t* moves, int32_t max_moves, int32_t* n_moves);

/* =============================================================================================
 * 2. Host tier memory (SMs stream host data straight into SMEM; no HBM staging)
 * ============================================================================================= */

/* Pinned, device-mapped, portable host allocation. *dev_ptr receives the device alias (== host
 * pointer under UVA). numa_node < 0: cudaHostAlloc (first-touch placement; write_combined allowed).
 * numa_node >= 0: anonymous pages bound to that node (mbind MPOL_BIND), faulted in, then
 * cudaHostRegister(Mapped | Portable): each GPU's host shard on the socket of its own link (SURVEY
 * §8(e)). Errors: DAK_EINVAL (bad arguments, mbind refused: no such node), DAK_EUNSUPPORTED
 * (write_combined with a node), DAK_ECUDA (CUDA / mmap failure). Free with dak_host_free. */
dak_status dak_host_alloc(size_t bytes, int32_t write_combined, int32_t numa_node, void** host_ptr, void** dev_ptr);
dak_status dak_host_free(void* host_ptr);
/* NUMA node of the current device's PCIe attachment (sysfs; -1 when the platform reports none). */
dak_status dak_device_numa_node(int32_t* node);

/* =============================================================================================
 * 2b. Congestion-control calibration (§3.3; SURVEY §8(f) rank 4 "online calibration")
 * ============================================================================================= */

/* Sweep of the calibration: n_host[i] host CTAs x window[j] x chunk_bytes host bytes in flight per
 * host CTA. Steady-state probe runs last duration_us; every sweep point times dak_linear (N = 8,
 * K = 7168, op_mb MiB of weights at the balanced ratio) end to end, median of reps chains of 8.
 * tolerance in [0, 1): the choice is the cheapest point within that fraction of the fastest. */
typedef struct {
  int32_t n_host[8];
  int32_t n_n_host;
  int32_t window[8];
  int32_t n_window;
  int32_t chunk_bytes;
  int32_t duration_us;
  int32_t reps;
  int32_t op_mb;      /* weight bytes of the end-to-end probe GEMV in MiB (0: 384) */
  double tolerance;
} dak_calib_opts;

/* Calibrated operating point: the launch configuration (dak_launch_cfg.n_cta_host and
 * host_inflight_kb = host_inflight_bytes / 1024) and the machine model of the planner (dak_hw:
 * hbm_bps = B_g and link_bps = B_h measured CONCURRENTLY at that point, host_latency_s = tau: one
 * chunk in flight, minus its transfer time at link_bps). hbm_alone_bps: every SM on HBM. */
typedef struct {
  int32_t n_cta_host;
  int32_t window;
  int64_t host_inflight_bytes;
  double hbm_bps;
  double link_bps;
  double hbm_alone_bps;
  double host_latency_s;
} dak_calib_result;

/* The choice (pure): table[i][j] = {HBM B/s, host B/s} of the end-to-end probe op at point
 * (n_host[i], window[j]) (each tier's bytes / the op's time): among the points whose aggregate (HBM +
 * host, summed in that order) is >= (1 - tolerance) x the best ("the exact SM allocation to the host
 * that maximizes end-to-end throughput"), the fewest host CTAs, then the smallest window
 * ("exactly enough SMs ... and avoid congestion"); ties: the first index. Errors: DAK_EINVAL. */
dak_status dak_calib_select(const double* table, int32_t n_n_host, int32_t n_window, const int32_t* n_host,
                            const int32_t* window, double tolerance, int32_t* best_i, int32_t* best_j);

/* The "lightweight parameter-sweeping profiler executed prior to kernel launch": measures
 * B_g (every SM on HBM), the saturated link rate and the link latency with steady-state probes (the
 * decode kernels' bulk-copy load path without the math, one CTA per SM), then times the split GEMV
 * at the balanced ratio r = B_h / (B_g + B_h) over opts' grid, on
 * hbm_buf (device; >= op_mb MiB + 1 MiB, and well above the 126 MB L2) and host_buf (pinned +
 * mapped; >= 16 chunks and the probe GEMV's host rows, ~1% of op_mb), fills *out and, when table !=
 * NULL, table[n_n_host][n_window][2] (each tier's bytes / the GEMV's time, B/s).
 * SETUP-TIME call: blocking, on an internal stream, not graph-capturable; allocates a small device
 * buffer. Errors: DAK_EINVAL (bad options / buffers), DAK_ECUDA. */
dak_status dak_calibrate(const void* hbm_buf, size_t hbm_bytes, const void* host_buf, size_t host_bytes,
                         const dak_calib_opts* opts, dak_calib_result* out, double* table);

/* =============================================================================================
 * 3. Split-source linear: y = act(x W^T + bias) + residual   (§3.1)
 *    W [M,K] is split along M: rows [0,h) in host memory, rows [h,M) in HBM (R7/R14).
 * ============================================================================================= */

/* Kernel-native weight layout ("DAK-KC"): a tier block of R rows is stored chunk-major,
 * [ceil(K/KC)][R][KC] bf16, each row's KC elements forming KC/64 atoms of 128 B whose 16-byte
 * chunks are XOR-swizzled by (row & 7) (bank-conflict-free ldmatrix / LDS.128). One k-chunk of
 * any contiguous row range is then ONE contiguous span -> one bulk copy per pipeline stage.
 * Requirements: K % 64 == 0, KC % 64 == 0, KC <= 2048. */
size_t dak_linear_packed_bytes(int64_t rows, int64_t K, int32_t kc);

/* Re-layout a row-major block src [rows, K] (bf16) into the DAK-KC layout at dst.
 * src/dst may be device or mapped-host pointers (the copy runs on the GPU, async on stream). */
dak_status dak_pack_linear(const void* src, int64_t rows, int64_t K, int32_t kc, void* dst, dak_stream_t stream);

/* Preferred KC for an op (chunk width so one stage of the per-CTA row range is ~16-48 KB). */
int32_t dak_linear_default_kc(int64_t M, int64_t K, int32_t n_ctas);
/* KC for the mma.sync decode path given the rows one CTA owns: the widest of {256, 128, 64}
 * dividing K whose stage (rows x KC) holds those rows within 48 KB and the path's accumulator
 * capacity: rows <= 96 -> 256, rows <= 192 -> 128, else 64. */
int32_t dak_linear_choose_kc(int64_t rows_per_cta, int64_t K);

#define DAK_ACT_NONE 0
#define DAK_ACT_RELU 1

typedef struct {
  int32_t n_cta_host;         /* CTAs that read the host tier (0: auto from calibration)       */
  int32_t n_cta_hbm;          /* CTAs that read HBM (0: SMs - n_cta_host)                      */
  int32_t window;             /* congestion window W: max in-flight host stages per CTA*/
                              /* (dak_attention: per warp; 0 with congestion_control: 512 KB of */
                              /* host tiles in flight over all host CTAs, >= 2 tiles per warp)  */
  int32_t stages;             /* SMEM ring depth for HBM CTAs (0: fill shared memory; attention: */
                              /* cap on ring slots per warp)                                     */
  int32_t congestion_control; /* 1: cap host CTAs / window as calibrated          */
  int32_t pdl;                /* 1: programmatic dependent launch (weights stream before the   */
                              /*    previous kernel finishes; x/residual read after it)        */
  int32_t force_path;         /* 0 auto, 1 CUDA-core FMA, 2 mma.sync, 3 tcgen05 (kc == 64),     */
                              /* 4 tcgen05 swapped operands (split-K decode form, N <= 128),    */
                              /* 5 CTA-pair tcgen05 GEMM (cta_group::2, 256-row pair tiles; auto */
                              /*   for a plain GEMM with h == 0 and N > 256; plain GEMM only)    */
  int32_t l2_policy;          /* 0: stream weights/KV with the L2 evict_first hint (they are   */
                              /*    read once per step), 1: no hint                              */
  int32_t cluster;            /* dak_linear: CTAs per thread-block cluster sharing ONE fetch of */
                              /* each x chunk by TMA multicast (P:L555-571 applied to the        */
                              /* operand every CTA reads); 0/1 off, 2 or 4. Same outputs bitwise */
                              /* N > 512 (tcgen05 groups of ceil(N/512) CTAs over the same rows): */
                              /* >= 2 makes each group one cluster whose rank 0 multicasts every  */
                              /* weight tile to the group: one HBM / link fetch per tile (Table 1)*/
  int32_t host_inflight_kb;   /* congestion control: host bytes in flight over all host CTAs, in KB */
                              /* (0: the built-in defaults, 256 KB linear / 512 KB attention;     */
                              /* dak_calibrate's host_inflight_bytes / 1024)                        */
} dak_launch_cfg;

typedef struct {
  const void* w_host;   /* DAK-KC packed rows [0,h)   (mapped host; may be NULL when h == 0)  */
  const void* w_hbm;    /* DAK-KC packed rows [h,M)   (device; may be NULL when h == M)       */
  int64_t M, K, h;      /* 0 <= h <= M                                                         */
  int32_t kc;           /* KC used to pack both tiers                                          */
  int32_t N;            /* batch columns, 1..64 (1..4096 on the tcgen05 path: kc == 64; N > 256 */
                        /* plain GEMM only: no ln_w / x_swiglu / stats_out)                  */
  const void* x;        /* [N, K] bf16 row-major, device                                       */
  void* y;              /* [N, M] bf16 row-major, device                                       */
  const void* bias;     /* [M] bf16 or NULL                                                    */
  const void* residual; /* [N, M] bf16 or NULL (added after the activation; may alias y)      */
  int32_t act;          /* DAK_ACT_*                                                           */
  int32_t reserved;
  dak_launch_cfg cfg;
  int64_t ldy;          /* elements between rows n of y and residual (0: M); lets q/k/v write   */
                        /* into one fused [N, (Hq+2Hkv)d] buffer                                */
  const void* l2_prefetch;   /* optional hint (NULL: none): device bytes the NEXT op reads first  */
  int64_t l2_prefetch_bytes; /* (multiple of 16). Once a CTA has issued its last weight copy, it  */
                             /* prefetches slice cta/grid of this span into L2, so the next op's  */
                             /* first stages hit L2 while this op drains. Never changes results.  */
  /* Fused pre-norm of x (OPT pre-LayerNorm; Llama RMSNorm). When ln_w != NULL the GEMV   */
  /* operand is bf16(((x - mu_n) * rstd_n) * ln_w + ln_b) -- exactly the dak_layernorm output --  */
  /* with mu_n, rstd_n = 1/sqrt(var_n + ln_eps) merged (Chan et al., fixed order) from ln_parts    */
  /* partial statistics ln_stats[part][N] = float4 (count, mean, M2, 0) written by the producer of  */
  /* x (stats_out of a dak_linear, or dak_embed / dak_row_stats). ln_rms = 1: RMSNorm (mu = 0,     */
  /* var = mean of squares, ln_b must be NULL). Tensor-core path only.                             */
  const void* ln_w;
  const void* ln_b;
  const float* ln_stats;
  int32_t ln_parts;
  int32_t ln_rms;
  float ln_eps;
  int32_t reserved2;
  /* Epilogue row statistics (nullable): CTA c writes float4 (count, mean, M2, 0) of its stored    */
  /* (bf16-rounded) outputs of row n to stats_out[c * N + n]; `grid` (dak_linear_query) parts.     */
  float* stats_out;
  /* SwiGLU operand (Llama MLP down projection): x is [N, 2K] = [gate | up] (row stride 2K) and the  */
  /* GEMV operand is bf16(silu(gate) * up), computed in fp32. Tensor-core path, no pre-norm.        */
  int32_t x_swiglu;
  int32_t reserved3;
  /* Workspace (device, nullable): lets the tcgen05 path split K when its 128-row tiles would be   */
  /* mostly empty (fp32 partials [splits][N][M], combined in fixed order by a second kernel).      */
  void* workspace;
  int64_t workspace_bytes;
} dak_linear_args;

/* Launch description (pure query; used by tests and the bench to attribute bytes). */
typedef struct {
  int32_t grid, n_cta_host, n_cta_hbm, threads;
  int32_t stages_hbm, window_host, smem_bytes, path; /* path: 1 FMA, 2 mma.sync               */
  int64_t rows_per_cta_host_max, rows_per_cta_hbm_max;
  int64_t hbm_bytes, host_bytes;                      /* algorithmic weight bytes per tier     */
  int32_t cluster;                                    /* CTAs sharing one x fetch (multicast)  */
  int32_t ksplit;                                     /* K splits (tcgen05 path, caller workspace); */
                                                      /* > 1 adds one split-K reduce launch     */
  int32_t host_gate;                                  /* split-K with congestion control: host   */
                                                      /* item CTAs streaming at once (0: no cap) */
  int32_t kblock;                                     /* split-K: rows per item (0: not split)   */
} dak_linear_launch_info;

dak_status dak_linear_query(const dak_linear_args* args, dak_linear_launch_info* info);

/* Workspace bytes the launch would use for split-K (0: none). Needs the device. */
size_t dak_linear_workspace_size(const dak_linear_args* args);

/* Row ownership of CTA `cta` (0 <= cta < grid): tier (0 HBM, 1 host) and [row_begin,row_end)
 * in global row numbering. Host CTAs split [0,h), HBM CTAs split [h,M), each into contiguous
 * ranges whose sizes differ by at most one row (8-row units on the tcgen05 path).
 * Split-K plans (ksplit > 1): CTA j of a tier owns the K split j % ksplit of the kblock-row block
 * j / ksplit of that tier (dak_linear_launch_info.kblock). N > 512 CTA groups: the group's rows. Pure query. */
dak_status dak_linear_cta_rows(const dak_linear_args* args, int32_t cta, int32_t* tier, int64_t* row_begin, int64_t* row_end);

/* Enqueue the split GEMV / skinny GEMM. */
dak_status dak_linear(const dak_linear_args* args, dak_stream_t stream);

/* A chain of split GEMVs in ONE persistent launch (one CTA per SM): each CTA walks the ops in
 * order with the row partition, arithmetic and epilogue of dak_linear's mma.sync path (outputs
 * bitwise equal to launching each op alone with cfg.force_path = 2 and the same kc / n_cta_host),
 * while its producer streams the next ops' weight stages into the same SMEM ring -- no per-op
 * drain and restart. An op whose x / residual / y overlaps an earlier op's buffers (x of op i = y of
 * op i-1 in a decode chain) reads x only after every CTA finished op i-1 (per-op counters in
 * `workspace`). Limits: 1 <= n_ops <= 16; every op has the same N (1..16) and kc; plain GEMV ops (no
 * ln_w / x_swiglu / stats_out / cluster; bias, ReLU, residual allowed); ops[0].cfg.pdl applies to
 * the launch; each op's n_cta_host / window / congestion_control / host_inflight_kb apply to it.
 * workspace: device, >= 4 * n_ops bytes, 16-byte aligned, ZERO-FILLED before the first call (each
 * call leaves it zeroed). Errors: DAK_EINVAL, DAK_EUNSUPPORTED, DAK_ECUDA. */
dak_status dak_linear_chain(const dak_linear_args* ops, int32_t n_ops, void* workspace, size_t workspace_bytes,
                            dak_stream_t stream);

/* =============================================================================================
 * 4. Split paged GQA decode attention  (P:L631 SplitK_FlashAttn; P:L386 decode attention)
 *    o[b, h] = softmax(scale * K_b q[b,h]) V_b over the tokens [0, seq_len[b]) of request b,
 *    kv head g = h / (Hq/Hkv); K_b, V_b gathered through block_table[b]; bit 31 of an entry
 *    selects the host pool, the low 31 bits index the page in that pool.
 * ============================================================================================= */

/* KV page layout ("DAK-PG"): a pool is [P][Hkv][page_size][d] bf16; each [page_size][d] block
 * stores the 16-byte chunk j of token row t at ((j>>3)<<3) | ((j&7) ^ (t&7)). Token slots of a
 * page beyond seq_len must hold finite values (pools are zero-initialised by their owner). */
dak_status dak_pack_kv_pages(const void* src, int64_t n_blocks, int32_t page_size, int32_t d, void* dst,
                             dak_stream_t stream);

typedef struct {
  const void* q;                /* [B, Hq, d] bf16, device                                      */
  void* out;                    /* [B, Hq, d] bf16, device                                      */
  const void* k_hbm;            /* DAK-PG pools in HBM (NULL if no HBM pages)                   */
  const void* v_hbm;
  const void* k_host;           /* DAK-PG pools in pinned mapped host memory (NULL if none)     */
  const void* v_host;
  const int32_t* block_table;   /* [B, max_pages] device; bit 31 = host tier                   */
  const int32_t* seq_lens;      /* [B] device, 1 <= seq_len <= max_pages*page_size              */
  int32_t B, Hq, Hkv, d;        /* d == 128; Hq % Hkv == 0; Hq/Hkv <= 8                         */
  int32_t page_size;            /* tokens per page, multiple of 16, <= 256                      */
  int32_t max_pages;            /* block-table row length                                       */
  int32_t chunk_pages;          /* split-KV chunk (pages); a chunk's tier = its first page's    */
  float scale;                  /* softmax scale; <= 0 means 1/sqrt(d) (SDPA default)          */
  void* workspace;              /* device, >= dak_attention_workspace_size bytes                */
  size_t workspace_bytes;
  dak_launch_cfg cfg;           /* n_cta_host, n_cta_hbm, window, stages, congestion_control,   */
                                /* pdl are honoured; force_path is ignored                      */
  int64_t q_row_stride;         /* elements between requests in q (0: Hq*d; fused QKV: (Hq+2Hkv)*d) */
  const void* k_new;            /* optional fused KV append (dak_kv_append in the same kernel): the */
  const void* v_new;            /* new token's k / v rows [B, Hkv, d] bf16 (row stride below) are  */
  int64_t kv_new_stride;        /* written at position seq_len - 1 into the pools (which must be   */
                                /* writable) and used for this step. NULL: the pools already hold */
                                /* the token (dak_kv_append ran). Stride 0: Hkv*d; 16-byte aligned */
} dak_attention_args;

/* With cfg.pdl, the block table, seq_lens and the KV rows of tokens < seq_len - 1 are read BEFORE
 * griddepcontrol.wait (they are step inputs / written by earlier steps), q and the row of the
 * newest token after it: the kernel immediately preceding may only produce q and that row. */

/* Pure query: workspace bytes (split-KV partials: B*Hkv*ceil(max_pages/chunk_pages)*(Hq/Hkv)*(d+1)*4). */
dak_status dak_attention_workspace_size(const dak_attention_args* args, size_t* bytes);

/* Enqueue split attention + the chunk combine (two kernels on `stream`). */
dak_status dak_attention(const dak_attention_args* args, dak_stream_t stream);

/* Decode KV write: the K/V rows of the new token of every (request, kv head) go to position
 * positions[b] of request b (page block_table[b][pos / page_size], row pos % page_size), in the
 * tier the block-table entry names. k_new, v_new: [B, Hkv*d] bf16 device rows, row_stride
 * elements apart (0: Hkv*d; rows of a fused QKV output: (Hq+2Hkv)*d). */
dak_status dak_kv_append(const void* k_new, const void* v_new, int64_t row_stride, const int32_t* block_table,
                         const int32_t* positions, int32_t B, int32_t Hkv, int32_t d, int32_t page_size,
                         int32_t max_pages, void* k_hbm, void* v_hbm, void* k_host, void* v_host, int32_t pdl,
                         dak_stream_t stream);

/* Carry out dak_kv_replace's moves on one layer's pools: page (all Hkv heads, K and V, DAK-PG
 * layout) of entry moves[2i] copied to entry moves[2i+1]. moves: device int32 [n_moves][2]. Pools as
 * of dak_attention_args, host pools pinned + mapped. Async on stream (graph-capturable); the
 * caller orders it after the step that last read the old table and before the first step that
 * reads the new one. Errors: DAK_EINVAL. */
dak_status dak_kv_migrate(const int32_t* moves, int32_t n_moves, int32_t Hkv, int32_t page_size, int32_t d, void* k_hbm,
                          void* v_hbm, void* k_host, void* v_host, dak_stream_t stream);

/* Llama decode KV write with rotary positions (BASELINE configs[2] model): for every request b,
 * rotate q (in place, all Hq heads) and k of the new token at positions[b] (rotate-half pairs
 * (i, i + d/2), angle pos / theta^(2i/d)), then write the rotated k and v rows into the pools at
 * positions[b] like dak_kv_append. qkv: [B, row_stride] bf16 rows holding q | k | v.
 * With pdl = 1, positions and block_table are read before the dependency wait: they must not be
 * written by the kernel launched just before (they are step inputs). */
dak_status dak_rope_kv_append(void* qkv, int64_t row_stride, int32_t B, int32_t Hq, int32_t Hkv, int32_t d,
                             const int32_t* positions, float rope_theta, const int32_t* block_table, int32_t page_size,
                             int32_t max_pages, void* k_hbm, void* v_hbm, void* k_host, void* v_host, int32_t pdl,
                             dak_stream_t stream);

/* Causal prefill attention over the same tier-split paged KV cache (P:L388
 * §3.2 "prefill ... arithmetic intensity O(L)": compute-bound at long L, the planner's Phase 2
 * regime, P:L429 / P:L453). Request b's T newest tokens sit at positions seq_lens[b] - T ..
 * seq_lens[b] - 1 and their K / V rows are already in the pools; query i attends keys
 * 0 .. seq_lens[b] - T + i (causal), kv head g = h / (Hq / Hkv):
 *   out[b, i, h] = softmax(scale * K_b[0 .. L-T+i] q[b, i, h]) V_b[0 .. L-T+i].
 * One CTA per (request, kv head, 128 query rows (token, head of the group)); 64-token K / V tiles
 * stream newest keys first from the tier each page's block-table entry names (bit 31 = host pool),
 * so the result is bitwise independent of the tier split. */
typedef struct {
  const void* q;                /* [B, T, Hq, d] bf16, device                                   */
  void* out;                    /* [B, T, Hq, d] bf16, device                                   */
  const void *k_hbm, *v_hbm;    /* DAK-PG pools in HBM (may be NULL if unused)                  */
  const void *k_host, *v_host;  /* DAK-PG pools in pinned mapped host memory (may be NULL)      */
  const int32_t* block_table;   /* [B, max_pages] device; bit 31 = host tier                   */
  const int32_t* seq_lens;      /* [B] device, T <= seq_len <= max_pages * page_size            */
  int32_t B, T, Hq, Hkv, d;     /* d == 128; Hq % Hkv == 0                                      */
  int32_t page_size;            /* multiple of 64 tokens                                        */
  int32_t max_pages;
  float scale;                  /* <= 0: 1/sqrt(d)                                              */
  dak_launch_cfg cfg;           /* stages (ring depth, 0: 6); n_cta_host = host streamer CTAs    */
  void* workspace;              /* device, >= dak_prefill_workspace_size, or NULL (see below)    */
  size_t workspace_bytes;
} dak_prefill_args;

/* Host tier (one tier per SM): with a workspace, cfg.n_cta_host (default 4) streamer CTAs
 * read every host page of the batch ONCE over the link into a device staging pool (newest pages
 * first) while the compute CTAs work newest-keys-first from HBM; a compute CTA reads a host-tier
 * tile from the staging pool once its page flag is up. Without a workspace every CTA reads host
 * tiles over the link itself: each host byte crosses the link once per query block of its
 * (request, kv head) -- Table 1's read amplification. Either way the result is the
 * same bits (keys are consumed newest first whatever their tier).
 * Errors: DAK_EINVAL (NULL / misaligned / non-positive sizes, Hq % Hkv, workspace too small),
 * DAK_EUNSUPPORTED (d != 128, page_size % 64). seq_lens are not checked on the host (device data). */
dak_status dak_prefill_workspace_size(const dak_prefill_args* args, size_t* bytes);
dak_status dak_prefill_attention(const dak_prefill_args* args, dak_stream_t stream);

/* =============================================================================================
 * 4b. Tensor-parallel combine (BASELINE north_star: TP over 8 x B200, NCCL over NVLink/NVSwitch)
 *     Row-parallel projections (o, down) leave a PARTIAL [rows, cols] output on every rank.
 * ============================================================================================= */

/* NCCL communicator (libnccl.so.2 bound at run time). dak_comm_unique_id writes 128 bytes on one
 * rank; the caller broadcasts them (e.g. torch.distributed) and every rank calls dak_comm_init. */
dak_status dak_comm_unique_id(void* id_out);
dak_status dak_comm_init(const void* id, int32_t rank, int32_t world, void** comm);
dak_status dak_comm_destroy(void* comm);

/* Ranks in the communicator (comm NULL: 1). */
dak_status dak_comm_size(void* comm, int32_t* world);

/* Column-parallel combine (Megatron column split: rank r computed output features
 * [r Ml, (r + 1) Ml) of y = x W^T, e.g. a TP-sharded GEMV of BASELINE configs[4]): recv [N, world*Ml]
 * bf16 row-major = the ranks' send [N, Ml] blocks side by side (ncclAllGather over NVLink, then one
 * re-layout kernel from NCCL's rank-major [world][N][Ml] in `scratch`; N == 1 or one rank: no
 * re-layout, scratch may be NULL). comm NULL: one rank (recv = send, copied unless aliased).
 * Ml % 8 == 0; 16-byte aligned device buffers. Errors: EINVAL, ENCCL, ECUDA. */
dak_status dak_allgather_cols(void* comm, const void* send, void* recv, void* scratch, int32_t N, int64_t Ml,
                              dak_stream_t stream);

/* partial (bf16 [rows, cols], device) is summed over the communicator in place (comm NULL: one
 * rank, no exchange), then x += partial (bf16 RNE) and, if stats_out != NULL, stats_out[r] =
 * float4 (cols, mean, M2, 0) of the new row r of x (a fused pre-norm's ln_stats, 1 part). */
/* As dak_allreduce_residual, then y_norm = RMSNorm(x) * norm_w (bf16 [rows, cols], the same
 * arithmetic as dak_rmsnorm) in the same kernel: the row-parallel o projection's combine and the
 * MLP pre-norm of a Llama layer in one launch. cols % 8 == 0, cols <= 16384, 16-byte aligned
 * pointers; y_norm may alias partial. Errors: EINVAL (NULL / misaligned), EUNSUPPORTED (cols). */
dak_status dak_allreduce_residual_rmsnorm(void* comm, void* partial, void* x, int32_t rows, int32_t cols,
                                          const void* norm_w, float eps, void* y_norm, int32_t pdl, dak_stream_t stream);
dak_status dak_allreduce_residual(void* comm, void* partial, void* x, int32_t rows, int32_t cols, float* stats_out,
                                  int32_t pdl, dak_stream_t stream);

/* NVLink-SHARP combine: a symmetric window of `bytes` (ncclMemAlloc +
 * ncclCommWindowRegister, bound to an NVSwitch multicast object) and an NCCL device communicator
 * with max_rows LSA barriers. Collective: every rank of `comm` calls it. *local_buf = this rank's
 * copy (device, 4 KB aligned): a row-parallel linear writes its bf16 partial there (dak_linear y).
 * Errors: DAK_EUNSUPPORTED (one rank, no multicast team, NCCL < 2.28: keep the ncclAllReduce
 * path), DAK_ENCCL, DAK_EINVAL. */
dak_status dak_nvls_create(void* comm, size_t bytes, int32_t max_rows, void** nvls, void** local_buf);
dak_status dak_nvls_destroy(void* nvls);
void* dak_nvls_local(void* nvls);
/* One kernel: LSA barrier; two-shot sum of the ranks' partials [rows, cols] at `offset` in the
 * window (rank r reduces rows i % world == r in the switch with multimem.ld_reduce, fp32
 * accumulation, and broadcasts them with multimem.st); barrier; x += sum (bf16 RNE); if norm_w:
 * y_norm = RMSNorm(x) * norm_w (as dak_allreduce_residual_rmsnorm). rows <= max_rows, cols % 8 == 0,
 * cols <= 16384. Every rank launches it for the same (offset, rows, cols). */
dak_status dak_nvls_residual_rmsnorm(void* nvls, size_t offset, void* x, int32_t rows, int32_t cols, const void* norm_w,
                                     float eps, void* y_norm, dak_stream_t stream);

/* =============================================================================================
 * 5. Decoder-layer decode step (the split operators as drop-in replacements inside
 *    the model; whole decode step CUDA-graph captured) and its glue kernels
 * ============================================================================================= */

/* y[r] = (x[r] - mean) * rsqrt(var + eps) * w + b over `cols`, fp32 statistics (b nullable). */
dak_status dak_layernorm(const void* x, const void* w, const void* b, void* y, int32_t rows, int32_t cols, float eps,
                         int32_t pdl, dak_stream_t stream);

/* x[b] = tok_emb[tokens[b]] + pos_emb[positions[b] + pos_offset]  (pos_emb/positions nullable;
 * OPT uses pos_offset 2). tokens/positions: device int32 [B]. */
dak_status dak_embed(const int32_t* tokens, const int32_t* positions, const void* tok_emb, const void* pos_emb,
                     int32_t B, int32_t hidden, int32_t pos_offset, void* x, float* stats_out, int32_t pdl,
                     dak_stream_t stream);

/* y[r] = x[r] / sqrt(mean(x[r]^2) + eps) * w  (RMSNorm, fp32 statistics). */
dak_status dak_rmsnorm(const void* x, const void* w, void* y, int32_t rows, int32_t cols, float eps, int32_t pdl,
                       dak_stream_t stream);

/* out[r, j] = bf16(silu(gu[r, j]) * gu[r, F + j]) for gu = [gate | up] rows of width 2F. */
dak_status dak_silu_mul(const void* gu, void* out, int32_t rows, int32_t F, int32_t pdl, dak_stream_t stream);

/* Row statistics for a fused pre-norm (dak_linear_args.ln_stats with ln_parts = 1):
 * stats_out[r] = float4 (cols, mean, M2 = sum (x - mean)^2, 0) over row r of x (bf16, row stride
 * ld elements, 0: cols), fp32, two-pass, fixed order. stats_out may be NULL in dak_embed. */
dak_status dak_row_stats(const void* x, int32_t rows, int32_t cols, int64_t ld, float* stats_out, int32_t pdl,
                         dak_stream_t stream);

/* One split weight of a layer: DAK-KC packed tiers (rows [0,h) host, [h,M) HBM), KC, bias. */
typedef struct {
  const void* w_host;
  const void* w_hbm;
  int64_t h;
  int32_t kc;
  int32_t n_cta_host;   /* 0: the layer cfg's value */
  const void* bias;     /* nullable */
} dak_weight;

typedef struct {
  int32_t model;                      /* DAK_MODEL_OPT | DAK_MODEL_LLAMA                      */
  int32_t B, hidden, n_heads, n_kv_heads, head_dim, ffn;
  float ln_eps;
  dak_weight qkv;                     /* fused [q;k;v] rows: (n_heads + 2 n_kv_heads) * head_dim */
  dak_weight o, up, down;             /* OPT: up = fc1 (ReLU), down = fc2                     */
  const void *ln1_w, *ln1_b, *ln2_w, *ln2_b;
  void* x;                            /* [B, hidden] bf16 residual stream, updated in place   */
  void* scratch;                      /* device, >= dak_layer_scratch_size                    */
  size_t scratch_bytes;
  void *k_hbm, *v_hbm, *k_host, *v_host;  /* this layer's KV pools (DAK-PG)                   */
  const int32_t* block_table;         /* [B, max_pages], bit 31 = host                         */
  const int32_t* positions;           /* [B] position of the new token                         */
  const int32_t* seq_lens;            /* [B] = positions + 1                                   */
  int32_t page_size, max_pages, chunk_pages;
  int32_t tp_rank, tp_size;           /* tensor-parallel rank / world (Llama)                    */
  int32_t x_prenormed;                /* Llama, fuse_norm 0: the scratch's normalised-x buffer   */
                                      /* already holds RMSNorm 1 of x (written by the previous   */
                                      /* layer's combine, see next_ln_w): skip that kernel       */
  dak_launch_cfg cfg;                 /* linear ops (pdl applies to every kernel)              */
  dak_launch_cfg attn_cfg;            /* attention                                             */
  int32_t split_qkv;                  /* 1: use q, k, v below instead of the fused qkv weight  */
  int32_t reserved2;
  dak_weight q, k, v;                 /* separate projections (rows Hq*d, Hkv*d, Hkv*d)         */
  int64_t l2_prefetch_bytes;          /* 0: off; else each linear warms this many leading bytes  */
                                      /* of the next linear's HBM tier (dak_linear_args hint)     */
  const void* next_w_hbm;             /* HBM tier of the op after this layer's last linear (the  */
  int64_t next_w_hbm_bytes;           /* next layer's q / qkv, or the LM head); nullable          */
  int32_t fuse_norm;                  /* 1: LN1 / LN2 fused into the consuming linears (no LN    */
                                      /*    kernels; x read raw, see dak_linear_args.ln_w)        */
  int32_t stats_in_parts;             /* partials in stats_in (dak_layer_stats_parts of the      */
  const float* stats_in;              /* previous layer, or 1 for dak_embed's statistics)        */
  float* stats_out;                   /* row statistics of this layer's output x (FC2 epilogue)  */
  /* Llama: n_heads / n_kv_heads / ffn are THIS rank's shard (heads n_heads*tp_rank ..); `up` is  */
  /* the fused [gate; up] weight (2 ffn rows), `down` takes the SwiGLU operand; ln*_w are RMSNorm */
  /* weights (ln*_b NULL); fuse_norm must be 1. With comm (required when tp_size > 1) o / down     */
  /* write partials that dak_allreduce_residual sums over `comm` before the residual add.         */
  float rope_theta;
  int32_t reserved4;
  void* comm;                         /* dak_comm_init communicator (required for tp_size > 1)  */
  const void* next_ln_w;              /* Llama, fuse_norm 0, comm set: the down projection's     */
                                      /* combine also writes RMSNorm(x) * next_ln_w (the next    */
                                      /* layer's RMSNorm 1) into the scratch for a next call with */
                                      /* x_prenormed = 1 and the same scratch; NULL: off          */
  void* nvls;                         /* Llama, fuse_norm 0, comm set: dak_nvls_create handle of */
                                      /* >= B * hidden * 2 bytes, B <= max_rows: o / down write    */
                                      /* their partials into its window and combine with          */
                                      /* dak_nvls_residual_rmsnorm (no ncclAllReduce); NULL: NCCL */
} dak_layer_args;

dak_status dak_layer_scratch_size(const dak_layer_args* args, size_t* bytes);
/* Enqueue one decode step of one layer: 8 kernels (LN, QKV, attention with the fused KV append + combine,
 * O + residual, LN, FC1 + ReLU, FC2 + residual). */
dak_status dak_layer(const dak_layer_args* args, dak_stream_t stream);
/* Number of statistics partials dak_layer writes to stats_out (the FC2 grid). Needs the device. */
dak_status dak_layer_stats_parts(const dak_layer_args* args, int32_t* parts);

#ifdef __cplusplus
}
#endif
#endif /* DAK_H_ */
