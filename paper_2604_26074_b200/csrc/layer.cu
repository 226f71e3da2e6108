// dak_layer — one decoder-layer decode step composed from the split-source operators
// (SplitK_GEMM / SplitK_FlashAttn as drop-in nn.Linear / SDPA replacements,
// the whole decode step captured in a CUDA graph). Glue kernels: LayerNorm, token+position
// embedding. OPT layer (pre-LN, biases, ReLU MLP, learned positions; P:L690 model family):
//
//   h = LN1(x); qkv = h Wqkv^T + b; append k, v at pos; a = attn(q, KV); x += a Wo^T + bo
//   h = LN2(x); f = relu(h W1^T + b1); x += f W2^T + b2
//
// Every weight is split host/HBM at its planned ratio. Each kernel is launched with
// programmatic dependent launch when cfg.pdl is set, so the next op's weight stream starts while
// the previous op drains (griddepcontrol.wait guards every dependent read).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace dak {
namespace layer {

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 4 + k] = t;
  }
}

constexpr int kLnThreads = 256;

__device__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < kLnThreads / 32; ++i) t += red[i];  // fixed order: deterministic
  __syncthreads();
  return t;
}

// y[r] = (x[r] - mean) / sqrt(var + eps) * w + b   (fp32 statistics, two-pass)
__global__ void __launch_bounds__(kLnThreads) layernorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ w,
                                                               const __nv_bfloat16* __restrict__ b,
                                                               __nv_bfloat16* __restrict__ y, int cols, float eps,
                                                               unsigned long long* tr, int rms) {
  __shared__ float red[kLnThreads / 32];
  tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  tstamp(tr, 1);
  const __nv_bfloat16* xr = x + (long long)blockIdx.x * cols;
  float s = 0.f;
  for (int c = threadIdx.x; c < cols; c += kLnThreads) s += __bfloat162float(xr[c]);
  const float mean = rms ? 0.f : block_sum(s, red) / (float)cols;  // RMSNorm: no centring
  float v = 0.f;
  for (int c = threadIdx.x; c < cols; c += kLnThreads) {
    const float d = __bfloat162float(xr[c]) - mean;
    v += d * d;
  }
  const float rstd = rsqrtf(block_sum(v, red) / (float)cols + eps);
  __nv_bfloat16* yr = y + (long long)blockIdx.x * cols;
  for (int c = threadIdx.x; c < cols; c += kLnThreads) {
    float t = (__bfloat162float(xr[c]) - mean) * rstd;
    t = t * __bfloat162float(w[c]) + (b ? __bfloat162float(b[c]) : 0.f);
    yr[c] = __float2bfloat16_rn(t);
  }
  tstamp(tr, 3);
}

// Vectorised form of layernorm_kernel for rows of cols % 8 == 0, cols <= 256 * 8 * kLnVec: each
// thread loads its 16-byte chunks once into registers (one HBM/L2 round trip per row instead of
// three scalar passes); RMSNorm skips the mean. Same per-element arithmetic as layernorm_kernel.
constexpr int kLnVec = 8;  // 16-byte chunks per thread
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
__global__ void __launch_bounds__(kLnThreads) layernorm_vec_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const __nv_bfloat16* __restrict__ w,
                                                                   const __nv_bfloat16* __restrict__ b,
                                                                   __nv_bfloat16* __restrict__ y, int cols, float eps,
                                                                   unsigned long long* tr, int rms) {
  __shared__ float red[kLnThreads / 32];
  tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  tstamp(tr, 1);
  const int nc = cols / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (long long)blockIdx.x * cols);
  uint4 raw[kLnVec];
#pragma unroll
  for (int i = 0; i < kLnVec; ++i) {
    const int c = threadIdx.x + i * kLnThreads;
    raw[i] = c < nc ? xr[c] : make_uint4(0u, 0u, 0u, 0u);
  }
  float mean = 0.f;
  if (!rms) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kLnVec; ++i) {
      float f[8];
      bf16x8_to_f32(raw[i], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += f[j];
    }
    mean = block_sum(s, red) / (float)cols;
  }
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < kLnVec; ++i) {
    if (threadIdx.x + i * kLnThreads < nc) {
      float f[8];
      bf16x8_to_f32(raw[i], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = f[j] - mean;
        v += d * d;
      }
    }
  }
  const float rstd = rsqrtf(block_sum(v, red) / (float)cols + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + (long long)blockIdx.x * cols);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int i = 0; i < kLnVec; ++i) {
    const int c = threadIdx.x + i * kLnThreads;
    if (c < nc) {
      float f[8], wf[8], bf[8];
      bf16x8_to_f32(raw[i], f);
      bf16x8_to_f32(wv[c], wf);
      if (b) bf16x8_to_f32(bv[c], bf);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = (f[j] - mean) * rstd * wf[j] + (b ? bf[j] : 0.f);
      yr[c] = f32_to_bf16x8(f);
    }
  }
  tstamp(tr, 3);
}

static bool ln_vec_ok(const void* x, const void* w, const void* b, const void* y, int cols) {
  return cols % 8 == 0 && cols <= kLnThreads * 8 * kLnVec && aligned16(x) && aligned16(w) && (!b || aligned16(b)) &&
         aligned16(y);
}

// (count, mean, M2) of one row held as one value per thread-slot, two-pass, fixed order
__device__ void row_stats_store(const float* v, int nv, int cols, float* red, float4* out) {
  float s = 0.f;
  for (int i = 0; i < nv; ++i) s += v[i];
  const float mean = block_sum(s, red) / (float)cols;
  float m2 = 0.f;
  for (int i = 0; i < nv; ++i) {
    const float d = v[i] - mean;
    m2 += d * d;
  }
  m2 = block_sum(m2, red);
  if (threadIdx.x == 0) *out = make_float4((float)cols, mean, m2, 0.f);
}

constexpr int kRowMax = 64;  // values per thread held in registers (cols <= 256 * 64)

// out[r, j] = bf16(silu(gu[r, j]) * gu[r, F + j])  (Llama MLP gate / up combine); 8 columns per
// thread (F % 8 == 0, 16-byte aligned rows), else one
// With part != nullptr, gate and up come from the producing linear's split-K fp32 partials
// (part[s][r][j], row stride 2F, gridDim.y rows): g = bf16(sum_s part) in split order, exactly the
// split-K reduce's value, then the same silu * up.
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int F,
                                unsigned long long* tr, int vec, const float* __restrict__ part, int S) {
  if (threadIdx.x == 0) tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  const __nv_bfloat16* g = gu + (long long)blockIdx.y * 2 * F;
  __nv_bfloat16* o = out + (long long)blockIdx.y * F;
  if (part) {  // F % 4 == 0: 4 columns per thread
    const long long split = (long long)gridDim.y * 2 * F;
    const float* pr = part + (long long)blockIdx.y * 2 * F;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F / 4; j += gridDim.x * blockDim.x) {
      float4 a = __ldcg(reinterpret_cast<const float4*>(pr) + j), u = __ldcg(reinterpret_cast<const float4*>(pr + F) + j);
      for (int s0 = 1; s0 < S; s0 += 4) {  // up to 4 splits' loads in flight, then summed in split order
        float4 ta[4], tu[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (s0 + q < S) {
            ta[q] = __ldcg(reinterpret_cast<const float4*>(pr + (s0 + q) * split) + j);
            tu[q] = __ldcg(reinterpret_cast<const float4*>(pr + (s0 + q) * split + F) + j);
          }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (s0 + q < S) {
            a.x += ta[q].x; a.y += ta[q].y; a.z += ta[q].z; a.w += ta[q].w;
            u.x += tu[q].x; u.y += tu[q].y; u.z += tu[q].z; u.w += tu[q].w;
          }
      }
      const float av[4] = {a.x, a.y, a.z, a.w}, uv[4] = {u.x, u.y, u.z, u.w};
      float r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float ga = __bfloat162float(__float2bfloat16_rn(av[i])), ua = __bfloat162float(__float2bfloat16_rn(uv[i]));
        r[i] = ga / (1.f + __expf(-ga)) * ua;
      }
      __nv_bfloat162 o0 = __floats2bfloat162_rn(r[0], r[1]), o1 = __floats2bfloat162_rn(r[2], r[3]);
      uint2 ob;
      ob.x = *reinterpret_cast<uint32_t*>(&o0);
      ob.y = *reinterpret_cast<uint32_t*>(&o1);
      reinterpret_cast<uint2*>(o)[j] = ob;
    }
  } else if (vec) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F / 8; j += gridDim.x * blockDim.x) {
      float a[8], u[8];
      bf16x8_to_f32(reinterpret_cast<const uint4*>(g)[j], a);
      bf16x8_to_f32(reinterpret_cast<const uint4*>(g + F)[j], u);
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = a[i] / (1.f + __expf(-a[i])) * u[i];
      reinterpret_cast<uint4*>(o)[j] = f32_to_bf16x8(a);
    }
  } else {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
      const float a = __bfloat162float(g[j]), u = __bfloat162float(g[F + j]);
      o[j] = __float2bfloat16_rn(a / (1.f + __expf(-a)) * u);
    }
  }
  if (threadIdx.x == 0) tstamp(tr, 3);
}

// x[b] = tok[tokens[b]] + pos[positions[b] + pos_offset]; optional row statistics of the stored x
__global__ void __launch_bounds__(kLnThreads) embed_kernel(const int* __restrict__ tokens, const int* __restrict__ positions,
                             const __nv_bfloat16* __restrict__ tok, const __nv_bfloat16* __restrict__ pos, int hidden,
                             int pos_offset, __nv_bfloat16* __restrict__ x, float4* __restrict__ stats,
                             unsigned long long* tr) {
  __shared__ float red[kLnThreads / 32];
  tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  const int b = blockIdx.x;
  const long long t = tokens[b];
  const long long p = positions ? (long long)positions[b] + pos_offset : -1;
  float v[kRowMax];
  int nv = 0;
  for (int c = threadIdx.x; c < hidden; c += kLnThreads) {
    float e = __bfloat162float(tok[t * hidden + c]);
    if (pos && p >= 0) e += __bfloat162float(pos[p * hidden + c]);
    const __nv_bfloat16 o = __float2bfloat16_rn(e);
    x[(long long)b * hidden + c] = o;
    if (nv < kRowMax) v[nv++] = __bfloat162float(o);
  }
  if (stats) row_stats_store(v, nv, hidden, red, stats + b);
  tstamp(tr, 3);
}

// Vectorised embed_kernel (hidden % 8 == 0, 16-byte aligned tables, hidden <= 256 * 8 * kLnVec):
// each thread gathers its 16-byte chunks of the token and position rows at once (one memory round
// trip instead of one per scalar), same per-element arithmetic; statistics two-pass from registers.
__global__ void __launch_bounds__(kLnThreads) embed_vec_kernel(const int* __restrict__ tokens, const int* __restrict__ positions,
                                 const __nv_bfloat16* __restrict__ tok, const __nv_bfloat16* __restrict__ pos, int hidden,
                                 int pos_offset, __nv_bfloat16* __restrict__ x, float4* __restrict__ stats,
                                 unsigned long long* tr) {
  __shared__ float red[kLnThreads / 32];
  tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  const int b = blockIdx.x;
  const long long t = tokens[b];
  const long long p = positions ? (long long)positions[b] + pos_offset : -1;
  const int nc = hidden / 8;
  const uint4* tr4 = reinterpret_cast<const uint4*>(tok + t * hidden);
  const uint4* pr4 = (pos && p >= 0) ? reinterpret_cast<const uint4*>(pos + p * hidden) : nullptr;
  uint4* xr = reinterpret_cast<uint4*>(x + (long long)b * hidden);
  float f[kLnVec][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kLnVec; ++i) {
    const int c = threadIdx.x + i * kLnThreads;
    if (c < nc) {
      float a[8];
      bf16x8_to_f32(tr4[c], a);
      if (pr4) {
        float q[8];
        bf16x8_to_f32(pr4[c], q);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += q[j];
      }
      const uint4 o = f32_to_bf16x8(a);
      xr[c] = o;
      bf16x8_to_f32(o, f[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += f[i][j];
    }
  }
  if (stats) {
    const float mean = block_sum(s, red) / (float)hidden;
    float m2 = 0.f;
#pragma unroll
    for (int i = 0; i < kLnVec; ++i)
      if (threadIdx.x + i * kLnThreads < nc) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = f[i][j] - mean;
          m2 += d * d;
        }
      }
    m2 = block_sum(m2, red);
    if (threadIdx.x == 0) stats[b] = make_float4((float)hidden, mean, m2, 0.f);
  }
  tstamp(tr, 3);
}

// stats[r] = (cols, mean, M2) of row r of x (bf16, row stride ld): the producer side of a fused pre-norm
__global__ void __launch_bounds__(kLnThreads) row_stats_kernel(const __nv_bfloat16* __restrict__ x, long long ld, int cols,
                                                              float4* __restrict__ stats) {
  __shared__ float red[kLnThreads / 32];
  grid_dep_launch();
  grid_dep_wait();
  float v[kRowMax];
  int nv = 0;
  for (int c = threadIdx.x; c < cols && nv < kRowMax; c += kLnThreads) v[nv++] = __bfloat162float(x[blockIdx.x * ld + c]);
  row_stats_store(v, nv, cols, red, stats + blockIdx.x);
}

static dak_status launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, cudaStream_t s, int pdl) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  return DAK_OK;
}

static inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

struct Scratch {
  size_t h, qkv, attn, f, f2, ws, stats, splitk, splitk_bytes, total, ws_bytes;
};
constexpr int kMaxParts = 1024;  // statistics partials (producer CTAs) a fused pre-norm merges

static dak_status scratch_layout(const dak_layer_args* a, Scratch* s) {
  if (a->model != DAK_MODEL_OPT && a->model != DAK_MODEL_LLAMA)
    return fail(DAK_EUNSUPPORTED, "dak_layer: model %d not in this build", a->model);
  if (a->B <= 0 || a->hidden <= 0 || a->n_heads <= 0 || a->n_kv_heads <= 0 || a->head_dim != 128 || a->ffn <= 0)
    return fail(DAK_EINVAL, "dak_layer: bad model sizes");
  const bool llama = a->model == DAK_MODEL_LLAMA;
  if (!llama && a->n_heads * a->head_dim != a->hidden) return fail(DAK_EINVAL, "dak_layer: n_heads * head_dim != hidden");
  if (a->tp_size < 1 || a->tp_rank < 0 || a->tp_rank >= a->tp_size) return fail(DAK_EINVAL, "dak_layer: bad tp rank / size");
  if (!llama && a->tp_size > 1) return fail(DAK_EUNSUPPORTED, "dak_layer: tensor parallelism is implemented for Llama");
  const size_t B = a->B;
  const size_t qkv_cols = (size_t)(a->n_heads + 2 * a->n_kv_heads) * a->head_dim;
  dak_attention_args at{};
  at.B = a->B; at.Hq = a->n_heads; at.Hkv = a->n_kv_heads; at.d = a->head_dim;
  at.page_size = a->page_size; at.max_pages = a->max_pages; at.chunk_pages = a->chunk_pages;
  at.cfg.n_cta_hbm = 1;
  size_t ws = 0;
  dak_status st = dak_attention_workspace_size(&at, &ws);
  if (st != DAK_OK) return st;
  const size_t attn_cols = (size_t)a->n_heads * a->head_dim;
  const size_t f_cols = (size_t)a->ffn * (llama ? 2 : 1);  // Llama: [gate | up]
  s->h = 0;
  s->qkv = align256(s->h + B * a->hidden * 2);  // h doubles as the TP partial buffer [B, hidden]
  s->attn = align256(s->qkv + B * qkv_cols * 2);
  s->f = align256(s->attn + B * attn_cols * 2);
  s->f2 = align256(s->f + B * f_cols * 2);  // Llama unfused: silu(gate) * up [B, ffn]
  s->ws = align256(s->f2 + (llama ? B * a->ffn * 2 : 0));
  s->ws_bytes = ws;
  s->stats = align256(s->ws + ws);
  // split-K partials of the tcgen05 path (batch > 16): <= 16 splits x B x the widest projection
  const size_t widest = std::max<size_t>(std::max<size_t>(qkv_cols, a->hidden), (size_t)a->ffn * (llama ? 2 : 1));
  s->splitk = align256(s->stats + (size_t)kMaxParts * B * 16);
  s->splitk_bytes = B > 16 ? 16 * B * widest * 4 : 0;
  s->total = s->splitk + s->splitk_bytes;
  return DAK_OK;
}

static dak_linear_args lin_args(const dak_weight& w, long long M, long long K, int N, const void* x, void* y,
                                const void* residual, int act, const dak_launch_cfg& cfg) {
  dak_linear_args l{};
  l.w_host = w.w_host;
  l.w_hbm = w.w_hbm;
  l.M = M; l.K = K; l.h = w.h; l.kc = w.kc; l.N = N;
  l.x = x; l.y = y; l.bias = w.bias; l.residual = residual; l.act = act;
  l.cfg = cfg;
  l.cfg.n_cta_host = w.n_cta_host > 0 ? w.n_cta_host : cfg.n_cta_host;
  return l;
}

// Llama decode layer (one tensor-parallel rank): RMSNorm fused into q/k/v and [gate; up], rotary +
// KV append, split attention, o (+ all-reduce) + residual, SwiGLU fused into down (+ all-reduce)
// + residual. 8 kernels per layer on one GPU (+2 NCCL all-reduces and 2 residual kernels at TP>1).
static dak_status llama_layer(const dak_layer_args* a, const Scratch& s, dak_stream_t stream) {
  // every linear of the layer may split K on the tcgen05 path: partials go to the scratch region
  void* const ws = s.splitk_bytes ? (char*)a->scratch + s.splitk : nullptr;
  const int64_t wsb = (int64_t)s.splitk_bytes;
  auto lin_args = [&](const dak_weight& w, long long M, long long K, int N, const void* x, void* y, const void* residual,
                      int act, const dak_launch_cfg& cfg) {
    dak_linear_args l = layer::lin_args(w, M, K, N, x, y, residual, act, cfg);
    l.workspace = ws;
    l.workspace_bytes = wsb;
    return l;
  };
  const bool fuse = a->fuse_norm != 0;
  if ((fuse && (!a->stats_in || a->stats_in_parts <= 0)) || a->ln1_b || a->ln2_b)
    return fail(DAK_EINVAL, "dak_layer (Llama): RMSNorm weights have no bias; fuse_norm needs stats_in");
  if (a->tp_size > 1 && !a->comm) return fail(DAK_EINVAL, "dak_layer (Llama): tp_size > 1 needs comm");
  char* sc = (char*)a->scratch;
  char* qkv = sc + s.qkv;
  void* attn = sc + s.attn;
  void* gu = sc + s.f;
  void* f2 = sc + s.f2;
  void* hbuf = sc + s.h;  // normalised x (unfused) -- the TP partial also lives here, never both at once
  // NVLS combine (unfused TP): the partials go into the symmetric window, one combine kernel
  const bool nv = a->nvls != nullptr && a->comm != nullptr && a->fuse_norm == 0;
  void* partial = nv ? dak_nvls_local(a->nvls) : sc + s.h;
  float* o_stats = (float*)(sc + s.stats);
  const int B = a->B, H = a->hidden, d = a->head_dim, Hq = a->n_heads, Hkv = a->n_kv_heads, F = a->ffn;
  const long long qkv_cols = (long long)(Hq + 2 * Hkv) * d;
  const int pdl = a->cfg.pdl;
  const bool tp = a->comm != nullptr;  // row-parallel partials + all-reduce (also usable at tp_size 1)
  cudaStream_t strm = (cudaStream_t)stream;
  dak_status st;
  // pre-norm: fused into the consuming linear (small batch: the per-CTA operand transform is
  // cheap), or one RMSNorm kernel into hbuf (large batch: every CTA would re-normalise all of x)
  auto rms = [&](dak_linear_args& l, const void* w, const float* stats, int parts) {
    l.x = a->x;
    l.ln_w = w; l.ln_b = nullptr; l.ln_rms = 1; l.ln_stats = stats; l.ln_parts = parts; l.ln_eps = a->ln_eps;
  };
  auto prenorm = [&](dak_linear_args& l, const void* w, const float* stats, int parts) -> dak_status {
    if (fuse) {
      rms(l, w, stats, parts);
      return DAK_OK;
    }
    l.x = hbuf;
    return dak_rmsnorm(a->x, w, hbuf, B, H, a->ln_eps, pdl, strm);
  };
  if (a->split_qkv) {  // q, k, v side by side into the [B, qkv_cols] buffer
    const long long rows[3] = {(long long)Hq * d, (long long)Hkv * d, (long long)Hkv * d};
    const dak_weight* w[3] = {&a->q, &a->k, &a->v};
    long long off = 0;
    for (int i = 0; i < 3; ++i) {
      dak_linear_args l = lin_args(*w[i], rows[i], H, B, a->x, qkv + off * 2, nullptr, DAK_ACT_NONE, a->cfg);
      l.ldy = qkv_cols;
      if (fuse) rms(l, a->ln1_w, a->stats_in, a->stats_in_parts);
      else if (i == 0 && (st = dak_rmsnorm(a->x, a->ln1_w, hbuf, B, H, a->ln_eps, pdl, strm)) != DAK_OK) return st;
      if (!fuse) l.x = hbuf;
      if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
      off += rows[i];
    }
  }
  int qkv_split = 1;  // split-K partials of the qkv projection, reduced inside the rotary/append kernel
  if (!a->split_qkv) {  // one fused [q; k; v] projection
    dak_linear_args l = lin_args(a->qkv, qkv_cols, H, B, a->x, qkv, nullptr, DAK_ACT_NONE, a->cfg);
    if (a->x_prenormed && !fuse) l.x = hbuf;  // RMSNorm 1 written by the previous layer's combine
    else if ((st = prenorm(l, a->ln1_w, a->stats_in, a->stats_in_parts)) != DAK_OK) return st;
    if ((st = linear_enqueue(&l, strm, true, &qkv_split)) != DAK_OK) return st;
  }
  if ((st = rope_kv_append_part(qkv, qkv_cols, B, Hq, Hkv, d, a->positions, a->rope_theta, a->block_table, a->page_size,
                                a->max_pages, a->k_hbm, a->v_hbm, a->k_host, a->v_host, pdl, strm,
                                qkv_split > 1 ? (const float*)ws : nullptr, qkv_split)) != DAK_OK)
    return st;
  dak_attention_args at{};
  at.q = qkv; at.out = attn;
  at.k_hbm = a->k_hbm; at.v_hbm = a->v_hbm; at.k_host = a->k_host; at.v_host = a->v_host;
  at.block_table = a->block_table; at.seq_lens = a->seq_lens;
  at.B = B; at.Hq = Hq; at.Hkv = Hkv; at.d = d;
  at.page_size = a->page_size; at.max_pages = a->max_pages; at.chunk_pages = a->chunk_pages;
  at.scale = 0.f;
  at.workspace = sc + s.ws; at.workspace_bytes = s.ws_bytes;
  at.cfg = a->attn_cfg;
  at.cfg.pdl = pdl;
  at.q_row_stride = qkv_cols;
  if ((st = dak_attention(&at, strm)) != DAK_OK) return st;
  // one-rank communicator, unfused combine: a split-K row-parallel linear leaves its fp32 partials
  // to the residual + RMSNorm kernel (no reduce launch; same arithmetic)
  int world = 1;
  if (tp && (st = dak_comm_size(a->comm, &world)) != DAK_OK) return st;
  const bool part_combine = tp && world == 1 && !nv && !fuse;
  int o_split = 1;
  // o projection: residual + statistics in the epilogue (1 rank), or partial -> all-reduce -> residual
  int o_parts = 1;
  if (part_combine) {
    dak_linear_args l = lin_args(a->o, H, (long long)Hq * d, B, attn, partial, nullptr, DAK_ACT_NONE, a->cfg);
    if ((st = linear_enqueue(&l, strm, true, &o_split)) != DAK_OK) return st;
  } else {
    dak_linear_args l = lin_args(a->o, H, (long long)Hq * d, B, attn, tp ? partial : a->x, tp ? nullptr : a->x,
                                 DAK_ACT_NONE, a->cfg);
    if (!tp && fuse) {
      dak_linear_launch_info info;
      if ((st = dak_linear_query(&l, &info)) != DAK_OK) return st;
      if (info.grid > kMaxParts) return fail(DAK_EUNSUPPORTED, "dak_layer: o grid %d > %d", info.grid, kMaxParts);
      o_parts = info.grid;
      l.stats_out = o_stats;
    }
    if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
  }
  // unfused TP: the combine kernel also writes RMSNorm 2 of the new x into hbuf (aliases partial)
  const bool norm2_done = tp && !fuse;
  if (norm2_done && nv) {
    if ((st = dak_nvls_residual_rmsnorm(a->nvls, 0, a->x, B, H, a->ln2_w, a->ln_eps, hbuf, strm)) != DAK_OK) return st;
  } else if (norm2_done && o_split > 1) {
    if ((st = residual_rmsnorm_part((const float*)ws, o_split, a->x, B, H, a->ln2_w, a->ln_eps, hbuf, pdl, strm)) != DAK_OK)
      return st;
  } else if (norm2_done) {
    if ((st = dak_allreduce_residual_rmsnorm(a->comm, partial, a->x, B, H, a->ln2_w, a->ln_eps, hbuf, pdl, strm)) != DAK_OK)
      return st;
  } else if (tp && (st = dak_allreduce_residual(a->comm, partial, a->x, B, H, fuse ? o_stats : nullptr, pdl, strm)) != DAK_OK) {
    return st;
  }
  int up_split = 1;  // split-K partials of [gate; up], reduced inside the silu * up kernel
  {  // [gate; up] after RMSNorm 2 -> gu [B, 2F]
    dak_linear_args l = lin_args(a->up, 2LL * F, H, B, a->x, gu, nullptr, DAK_ACT_NONE, a->cfg);
    if (norm2_done) l.x = hbuf;
    else if ((st = prenorm(l, a->ln2_w, o_stats, o_parts)) != DAK_OK) return st;
    if ((st = linear_enqueue(&l, strm, !fuse, &up_split)) != DAK_OK) return st;
  }
  {  // down: the SwiGLU operand fused (small batch) or one silu * up kernel (large batch)
    dak_linear_args l = lin_args(a->down, H, F, B, fuse ? gu : f2, tp ? partial : a->x, tp ? nullptr : a->x,
                                 DAK_ACT_NONE, a->cfg);
    if (fuse) l.x_swiglu = 1;
    else if ((st = silu_mul_part(gu, f2, B, F, pdl, strm, up_split > 1 ? (const float*)ws : nullptr, up_split)) != DAK_OK)
      return st;
    if (!tp && fuse) l.stats_out = a->stats_out;
    int down_split = 1;
    if ((st = linear_enqueue(&l, strm, part_combine && a->next_ln_w, &down_split)) != DAK_OK) return st;
    if (part_combine && a->next_ln_w && down_split > 1) {
      if ((st = residual_rmsnorm_part((const float*)ws, down_split, a->x, B, H, a->next_ln_w, a->ln_eps, hbuf, pdl, strm)) !=
          DAK_OK)
        return st;
    } else if (nv) {  // NVLS: one kernel (the next layer's RMSNorm 1 too when given)
      if ((st = dak_nvls_residual_rmsnorm(a->nvls, 0, a->x, B, H, a->next_ln_w, a->ln_eps, hbuf, strm)) != DAK_OK) return st;
    } else if (tp && !fuse && a->next_ln_w) {  // the next layer's RMSNorm 1 in the same combine kernel
      if ((st = dak_allreduce_residual_rmsnorm(a->comm, partial, a->x, B, H, a->next_ln_w, a->ln_eps, hbuf, pdl, strm)) != DAK_OK)
        return st;
    } else if (tp && (st = dak_allreduce_residual(a->comm, partial, a->x, B, H, fuse ? a->stats_out : nullptr, pdl, strm)) != DAK_OK) {
      return st;
    }
  }
  return DAK_OK;
}

}  // namespace layer
}  // namespace dak

using namespace dak;

extern "C" {

dak_status dak_layernorm(const void* x, const void* w, const void* b, void* y, int32_t rows, int32_t cols, float eps,
                         int32_t pdl, dak_stream_t stream) {
  if (!x || !w || !y || rows <= 0 || cols <= 0) return fail(DAK_EINVAL, "dak_layernorm: bad arguments");
  const __nv_bfloat16* xp = (const __nv_bfloat16*)x;
  const __nv_bfloat16* wp = (const __nv_bfloat16*)w;
  const __nv_bfloat16* bp = (const __nv_bfloat16*)b;
  __nv_bfloat16* yp = (__nv_bfloat16*)y;
  int c = cols;
  unsigned long long* tr = trace_slot(DAK_KIND_LAYERNORM, rows, cols, rows);
  int rms = 0;
  void* args[] = {&xp, &wp, &bp, &yp, &c, &eps, &tr, &rms};
  const bool vec = layer::ln_vec_ok(xp, wp, bp, yp, cols);
  return layer::launch_pdl(vec ? (const void*)layer::layernorm_vec_kernel : (const void*)layer::layernorm_kernel,
                           dim3(rows), dim3(layer::kLnThreads), args, (cudaStream_t)stream, pdl);
}

dak_status dak_rmsnorm(const void* x, const void* w, void* y, int32_t rows, int32_t cols, float eps, int32_t pdl,
                       dak_stream_t stream) {
  if (!x || !w || !y || rows <= 0 || cols <= 0) return fail(DAK_EINVAL, "dak_rmsnorm: bad arguments");
  const __nv_bfloat16* xp = (const __nv_bfloat16*)x;
  const __nv_bfloat16* wp = (const __nv_bfloat16*)w;
  const __nv_bfloat16* bp = nullptr;
  __nv_bfloat16* yp = (__nv_bfloat16*)y;
  int c = cols;
  unsigned long long* tr = trace_slot(DAK_KIND_LAYERNORM, rows, cols, rows);
  int rms = 1;
  void* args[] = {&xp, &wp, &bp, &yp, &c, &eps, &tr, &rms};
  const bool vec = layer::ln_vec_ok(xp, wp, bp, yp, cols);
  return layer::launch_pdl(vec ? (const void*)layer::layernorm_vec_kernel : (const void*)layer::layernorm_kernel,
                           dim3(rows), dim3(layer::kLnThreads), args, (cudaStream_t)stream, pdl);
}

dak_status dak_silu_mul(const void* gu, void* out, int32_t rows, int32_t F, int32_t pdl, dak_stream_t stream) {
  return dak::silu_mul_part(gu, out, rows, F, pdl, stream, nullptr, 1);
}

dak_status dak_embed(const int32_t* tokens, const int32_t* positions, const void* tok_emb, const void* pos_emb,
                     int32_t B, int32_t hidden, int32_t pos_offset, void* x, float* stats_out, int32_t pdl,
                     dak_stream_t stream) {
  if (!tokens || !tok_emb || !x || B <= 0 || hidden <= 0) return fail(DAK_EINVAL, "dak_embed: bad arguments");
  if (hidden > layer::kLnThreads * layer::kRowMax) return fail(DAK_EUNSUPPORTED, "dak_embed: hidden > %d", layer::kLnThreads * layer::kRowMax);
  if (stats_out && !aligned16(stats_out)) return fail(DAK_EINVAL, "dak_embed: stats_out must be 16-byte aligned");
  const int* tp = tokens;
  const int* pp = positions;
  const __nv_bfloat16* te = (const __nv_bfloat16*)tok_emb;
  const __nv_bfloat16* pe = (const __nv_bfloat16*)pos_emb;
  int h = hidden, off = pos_offset;
  __nv_bfloat16* xp = (__nv_bfloat16*)x;
  float4* sp = (float4*)stats_out;
  unsigned long long* tr = trace_slot(DAK_KIND_EMBED, B, hidden, B);
  void* args[] = {&tp, &pp, &te, &pe, &h, &off, &xp, &sp, &tr};
  const bool vec = hidden % 8 == 0 && hidden <= layer::kLnThreads * 8 * layer::kLnVec && aligned16(tok_emb) &&
                   (!pos_emb || aligned16(pos_emb)) && aligned16(x);
  return layer::launch_pdl(vec ? (const void*)layer::embed_vec_kernel : (const void*)layer::embed_kernel, dim3(B),
                           dim3(layer::kLnThreads), args, (cudaStream_t)stream, pdl);
}

dak_status dak_row_stats(const void* x, int32_t rows, int32_t cols, int64_t ld, float* stats_out, int32_t pdl,
                         dak_stream_t stream) {
  if (!x || !stats_out || rows <= 0 || cols <= 0) return fail(DAK_EINVAL, "dak_row_stats: bad arguments");
  if (cols > layer::kLnThreads * layer::kRowMax) return fail(DAK_EUNSUPPORTED, "dak_row_stats: cols > %d", layer::kLnThreads * layer::kRowMax);
  if (!aligned16(stats_out)) return fail(DAK_EINVAL, "dak_row_stats: stats_out must be 16-byte aligned");
  const __nv_bfloat16* xp = (const __nv_bfloat16*)x;
  long long l = ld > 0 ? ld : cols;
  int c = cols;
  float4* sp = (float4*)stats_out;
  void* args[] = {&xp, &l, &c, &sp};
  return layer::launch_pdl((const void*)layer::row_stats_kernel, dim3(rows), dim3(layer::kLnThreads), args,
                           (cudaStream_t)stream, pdl);
}

dak_status dak_layer_scratch_size(const dak_layer_args* a, size_t* bytes) {
  if (!a || !bytes) return fail(DAK_EINVAL, "dak_layer_scratch_size: NULL");
  layer::Scratch s;
  dak_status st = layer::scratch_layout(a, &s);
  if (st != DAK_OK) return st;
  *bytes = s.total;
  return DAK_OK;
}

dak_status dak_layer(const dak_layer_args* a, dak_stream_t stream) {
  if (!a) return fail(DAK_EINVAL, "dak_layer: NULL");
  layer::Scratch s;
  dak_status st = layer::scratch_layout(a, &s);
  if (st != DAK_OK) return st;
  if (!a->x || !a->scratch || a->scratch_bytes < s.total) return fail(DAK_EINVAL, "dak_layer: x / scratch missing or too small");
  const bool fuse = a->fuse_norm != 0;
  if (fuse && (!a->stats_in || a->stats_in_parts <= 0))
    return fail(DAK_EINVAL, "dak_layer: fuse_norm needs stats_in / stats_in_parts (row statistics of x)");
  if (a->model == DAK_MODEL_LLAMA) return layer::llama_layer(a, s, stream);
  char* sc = (char*)a->scratch;
  void* h = sc + s.h;
  char* qkv = sc + s.qkv;
  void* attn = sc + s.attn;
  void* f = sc + s.f;
  float* o_stats = (float*)(sc + s.stats);
  void* const ws = s.splitk_bytes ? sc + s.splitk : nullptr;
  const int64_t wsb = (int64_t)s.splitk_bytes;
  auto lin_args = [&](const dak_weight& w, long long M, long long K, int N, const void* x, void* y, const void* residual,
                      int act, const dak_launch_cfg& cfg) {
    dak_linear_args l = layer::lin_args(w, M, K, N, x, y, residual, act, cfg);
    l.workspace = ws;
    l.workspace_bytes = wsb;
    return l;
  };
  const int B = a->B, H = a->hidden, d = a->head_dim, Hq = a->n_heads, Hkv = a->n_kv_heads;
  const long long qkv_cols = (long long)(Hq + 2 * Hkv) * d;
  const int pdl = a->cfg.pdl;
  cudaStream_t strm = (cudaStream_t)stream;
  // L2 warm-up chain: every linear prefetches the leading bytes of the next linear's HBM tier
  const long long pfb = a->l2_prefetch_bytes;
  auto pf = [&](dak_linear_args& l, const dak_weight& w, long long rows, long long K) {
    const long long avail = (rows - w.h) * K * 2;
    if (pfb <= 0 || !w.w_hbm || avail <= 0) return;
    l.l2_prefetch = w.w_hbm;
    l.l2_prefetch_bytes = std::min(pfb, avail) & ~15LL;
  };
  // pre-norm: either a LayerNorm kernel into h, or fused into the consuming linears (x read raw)
  auto norm = [&](dak_linear_args& l, const void* w, const void* b, const float* stats, int parts) {
    l.x = a->x;
    l.ln_w = w; l.ln_b = b; l.ln_stats = stats; l.ln_parts = parts; l.ln_eps = a->ln_eps;
  };

  if (!fuse && (st = dak_layernorm(a->x, a->ln1_w, a->ln1_b, h, B, H, a->ln_eps, pdl, strm)) != DAK_OK) return st;
  dak_linear_args l;
  if (a->split_qkv) {  // q, k, v written side by side into the fused [B, qkv_cols] buffer
    const long long rows[3] = {(long long)Hq * d, (long long)Hkv * d, (long long)Hkv * d};
    const dak_weight* w[3] = {&a->q, &a->k, &a->v};
    long long off = 0;
    for (int i = 0; i < 3; ++i) {
      l = lin_args(*w[i], rows[i], H, B, h, qkv + off * 2, nullptr, DAK_ACT_NONE, a->cfg);
      l.ldy = qkv_cols;
      if (fuse) norm(l, a->ln1_w, a->ln1_b, a->stats_in, a->stats_in_parts);
      if (i < 2) pf(l, *w[i + 1], rows[i + 1], H);
      else pf(l, a->o, H, (long long)Hq * d);
      if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
      off += rows[i];
    }
  } else {
    l = lin_args(a->qkv, qkv_cols, H, B, h, qkv, nullptr, DAK_ACT_NONE, a->cfg);
    if (fuse) norm(l, a->ln1_w, a->ln1_b, a->stats_in, a->stats_in_parts);
    pf(l, a->o, H, (long long)Hq * d);
    if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
  }
  // the KV append (new token's k, v at position seq_len - 1) is fused into the attention kernel
  dak_attention_args at{};
  at.k_new = qkv + (size_t)Hq * d * 2;
  at.v_new = qkv + (size_t)(Hq + Hkv) * d * 2;
  at.kv_new_stride = qkv_cols;
  at.q = qkv; at.out = attn;
  at.k_hbm = a->k_hbm; at.v_hbm = a->v_hbm; at.k_host = a->k_host; at.v_host = a->v_host;
  at.block_table = a->block_table; at.seq_lens = a->seq_lens;
  at.B = B; at.Hq = Hq; at.Hkv = Hkv; at.d = d;
  at.page_size = a->page_size; at.max_pages = a->max_pages; at.chunk_pages = a->chunk_pages;
  at.scale = 0.f;
  at.workspace = sc + s.ws; at.workspace_bytes = s.ws_bytes;
  at.cfg = a->attn_cfg;
  at.cfg.pdl = pdl;
  at.q_row_stride = qkv_cols;
  if ((st = dak_attention(&at, strm)) != DAK_OK) return st;
  l = lin_args(a->o, H, (long long)Hq * d, B, attn, a->x, a->x, DAK_ACT_NONE, a->cfg);
  pf(l, a->up, a->ffn, H);
  int o_parts = 0;
  if (fuse) {
    dak_linear_launch_info info;
    if ((st = dak_linear_query(&l, &info)) != DAK_OK) return st;
    if (info.grid > layer::kMaxParts) return fail(DAK_EUNSUPPORTED, "dak_layer: o-projection grid %d > %d", info.grid, layer::kMaxParts);
    o_parts = info.grid;
    l.stats_out = o_stats;
  }
  if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
  if (!fuse && (st = dak_layernorm(a->x, a->ln2_w, a->ln2_b, h, B, H, a->ln_eps, pdl, strm)) != DAK_OK) return st;
  l = lin_args(a->up, a->ffn, H, B, h, f, nullptr, DAK_ACT_RELU, a->cfg);
  if (fuse) norm(l, a->ln2_w, a->ln2_b, o_stats, o_parts);
  pf(l, a->down, H, a->ffn);
  if ((st = dak_linear(&l, strm)) != DAK_OK) return st;
  l = lin_args(a->down, H, a->ffn, B, f, a->x, a->x, DAK_ACT_NONE, a->cfg);
  if (pfb > 0 && a->next_w_hbm && a->next_w_hbm_bytes > 0) {
    l.l2_prefetch = a->next_w_hbm;
    l.l2_prefetch_bytes = std::min(pfb, (long long)a->next_w_hbm_bytes) & ~15LL;
  }
  l.stats_out = a->stats_out;
  return dak_linear(&l, strm);
}

dak_status dak_layer_stats_parts(const dak_layer_args* a, int32_t* parts) {
  if (!a || !parts) return fail(DAK_EINVAL, "dak_layer_stats_parts: NULL");
  if (a->model == DAK_MODEL_LLAMA && a->comm) {  // written by dak_allreduce_residual: 1 per row
    *parts = 1;
    return DAK_OK;
  }
  dak_linear_args l = layer::lin_args(a->down, a->hidden, a->ffn, a->B, a->x, a->x, a->x, DAK_ACT_NONE, a->cfg);
  dak_linear_launch_info info;
  dak_status st = dak_linear_query(&l, &info);
  if (st != DAK_OK) return st;
  *parts = info.grid;
  return DAK_OK;
}

}  // extern "C"

dak_status dak::silu_mul_part(const void* gu, void* out, int32_t rows, int32_t F, int32_t pdl, void* stream,
                              const float* part, int32_t S) {
  if ((!gu && !part) || !out || rows <= 0 || F <= 0) return fail(DAK_EINVAL, "dak_silu_mul: bad arguments");
  if (part && (F % 4 || !aligned16(part) || ((uintptr_t)out & 7) || S < 1))
    return fail(DAK_EINVAL, "dak_silu_mul: split-K partials need F %% 4 == 0 and aligned buffers");
  const __nv_bfloat16* gp = (const __nv_bfloat16*)gu;
  __nv_bfloat16* op = (__nv_bfloat16*)out;
  int f = F;
  unsigned long long* tr = trace_slot(DAK_KIND_SILU, rows, F, rows);
  int vec = F % 8 == 0 && aligned16(gu) && aligned16(out);
  int s = S;
  void* args[] = {&gp, &op, &f, &tr, &vec, &part, &s};
  const int per = part ? F / 4 : vec ? F / 8 : F;
  const int bx = (per + 255) / 256 < 8 ? (per + 255) / 256 : 8;
  return layer::launch_pdl((const void*)layer::silu_mul_kernel, dim3(bx, rows), dim3(256), args, (cudaStream_t)stream, pdl);
}
