// Tensor-parallel combine for row-parallel projections (BASELINE north_star: TP over 8 x B200).
//
// Megatron layout: q/k/v/gate/up are split by output rows (heads / FFN rows, no exchange), o and
// down by input columns, so each rank holds a PARTIAL [B, H] output that is summed over ranks
// (NCCL all-reduce over NVLink / NVSwitch) before the residual add. dak_allreduce_residual does the
// all-reduce in place and then x += sum (bf16 RNE) and the row statistics a fused pre-norm of the
// next op consumes (one part per row). NCCL is bound at run time (dlopen of libnccl.so.2, the one
// torch already loaded), so the library loads and the single-GPU path runs without NCCL.
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "common.h"

namespace dak {
namespace tp {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

static dak_status nccl(Nccl** out) {
  static Nccl n;
  if (!n.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(DAK_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
    n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(h, "ncclCommInitRank");
    n.comm_destroy = (decltype(n.comm_destroy))dlsym(h, "ncclCommDestroy");
    n.all_reduce = (decltype(n.all_reduce))dlsym(h, "ncclAllReduce");
    n.error_string = (decltype(n.error_string))dlsym(h, "ncclGetErrorString");
    n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
    n.comm_count = (decltype(n.comm_count))dlsym(h, "ncclCommCount");
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce || !n.error_string || !n.all_gather ||
        !n.comm_count)
      return fail(DAK_ENCCL, "libnccl.so.2 lacks a required symbol");
    n.h = h;
  }
  *out = &n;
  return DAK_OK;
}

#define DAK_NCCL_TRY(n, expr)                                                                     \
  do {                                                                                           \
    ncclResult_t r__ = (expr);                                                                   \
    if (r__ != ncclSuccess) return fail(DAK_ENCCL, "%s failed: %s", #expr, (n)->error_string(r__)); \
  } while (0)

__device__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];  // fixed order
  __syncthreads();
  return t;
}

constexpr int kThreads = 256;
constexpr int kPer = 64;  // values per thread (cols <= 16384)

// x[r] += partial[r] (bf16 RNE); stats[r] = (cols, mean, M2) of the new x row (two-pass)
__global__ void __launch_bounds__(kThreads) residual_stats_kernel(const __nv_bfloat16* __restrict__ partial,
                                                                  __nv_bfloat16* __restrict__ x, int cols,
                                                                  float4* __restrict__ stats) {
  __shared__ float red[kThreads / 32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long base = (long long)blockIdx.x * cols;
  float v[kPer];
  int nv = 0;
  float s = 0.f;
#pragma unroll 4
  for (int c = threadIdx.x; c < cols; c += kThreads) {
    const __nv_bfloat16 o = __float2bfloat16_rn(__bfloat162float(x[base + c]) + __bfloat162float(partial[base + c]));
    x[base + c] = o;
    const float f = __bfloat162float(o);
    if (nv < kPer) v[nv++] = f;
    s += f;
  }
  if (!stats) return;
  const float mean = block_sum(s, red) / (float)cols;
  float m2 = 0.f;
  for (int i = 0; i < nv; ++i) {
    const float d = v[i] - mean;
    m2 += d * d;
  }
  m2 = block_sum(m2, red);
  if (threadIdx.x == 0) stats[blockIdx.x] = make_float4((float)cols, mean, m2, 0.f);
}

// Vectorised residual_stats_kernel (cols % 8 == 0, 16-byte aligned rows): chunks held in registers,
// the same per-element arithmetic; statistics two-pass from registers (fixed order).
__global__ void __launch_bounds__(kThreads) residual_stats_vec_kernel(const __nv_bfloat16* __restrict__ partial,
                                                                      __nv_bfloat16* __restrict__ x, int cols,
                                                                      float4* __restrict__ stats) {
  __shared__ float red[kThreads / 32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int nc = cols / 8;
  const long long base = (long long)blockIdx.x * nc;
  uint4* xr = reinterpret_cast<uint4*>(x) + base;
  const uint4* pr = reinterpret_cast<const uint4*>(partial) + base;
  float f[8][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = threadIdx.x + i * kThreads;
    if (c < nc) {
      const uint4 a = xr[c], b = pr[c];
      const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* bh = reinterpret_cast<const __nv_bfloat162*>(&b);
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 u = __bfloat1622float2(ah[j]), v = __bfloat1622float2(bh[j]);
        oh[j] = __floats2bfloat162_rn(u.x + v.x, u.y + v.y);
        const float2 r = __bfloat1622float2(oh[j]);
        f[i][2 * j] = r.x;
        f[i][2 * j + 1] = r.y;
        s += r.x + r.y;
      }
      xr[c] = o;
    }
  }
  if (!stats) return;
  const float mean = block_sum(s, red) / (float)cols;
  float m2 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (threadIdx.x + i * kThreads < nc) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = f[i][j] - mean;
        m2 += d * d;
      }
    }
  m2 = block_sum(m2, red);
  if (threadIdx.x == 0) stats[blockIdx.x] = make_float4((float)cols, mean, m2, 0.f);
}

// x[r] += partial[r] (bf16 RNE), then y[r] = bf16(x[r] * rstd * w) with rstd = 1/sqrt(mean(x^2) + eps)
// (RMSNorm of the new row: the same arithmetic as dak_rmsnorm, fused so the MLP pre-norm needs no
// launch of its own). y may alias partial (each thread reads its own chunks before it writes).
// part != nullptr (one rank): the row-parallel linear's split-K partials are reduced here instead of
// by its reduce kernel -- partial = bf16(sum_s part[s][r][c]) in split order, the arithmetic of
// splitk_reduce_kernel without bias / activation -- so the combine costs no extra launch.
//
// A row is split over a cluster of `cpr` CTAs (16-byte chunks [crank * per, ...)), each thread
// holding V chunks in registers: every load of a thread (x, the S partials) is issued before the
// first use -- one L2 round trip -- and the norm weight, a parameter, is loaded before the
// dependency wait. The row's sum of squares: per thread, warp shuffle, warps in order, then the
// cluster's CTA sums in rank order through distributed shared memory (every CTA adds the same
// values in the same order: the same rstd). A one-CTA-per-row form spent ~9 us per launch on
// dependent load round trips over 64 SMs (profiles/r02/step_launches_llama3-70b-tp8-b64-ctx4096.txt).
constexpr int kVec = 8;    // max 16-byte chunks per thread
constexpr int kMaxCpr = 8; // max CTAs per row (portable cluster size)
__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 4 + k] = t;
  }
}
__device__ __forceinline__ void add4(float4& a, const float4 c) {
  a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
}
template <int V>
__global__ void __launch_bounds__(kThreads) residual_rmsnorm_kernel(const __nv_bfloat16* partial,
                                                                    __nv_bfloat16* __restrict__ x, int cols,
                                                                    const __nv_bfloat16* __restrict__ w, float eps,
                                                                    __nv_bfloat16* y, const float* part, int S, int rows,
                                                                    int cpr, unsigned long long* tr) {
  __shared__ float red[kThreads / 32];
  __shared__ float cta_sum;
  tstamp(tr, 0);
  const int nc = cols / 8;
  const int crank = (int)blockIdx.x % cpr, row = (int)blockIdx.x / cpr;
  const int per = (nc + cpr - 1) / cpr;
  const int c0 = crank * per, c1 = min(nc, c0 + per);
  const long long base = (long long)row * nc;
  uint4 wv[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {  // parameters: loaded while the producing kernel drains
    const int c = c0 + threadIdx.x + i * kThreads;
    if (c < c1) wv[i] = __ldg(reinterpret_cast<const uint4*>(w) + c);
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tstamp(tr, 1);
  uint4* xr = reinterpret_cast<uint4*>(x) + base;
  uint4 xa[V], pb[V];
  float4 lo[V], hi[V];
  const long long plane = (long long)rows * cols;
#pragma unroll
  for (int i = 0; i < V; ++i) {  // every load of the thread first: one round trip
    const int c = c0 + threadIdx.x + i * kThreads;
    if (c < c1) {
      xa[i] = xr[c];
      if (part) {
        const float* q = part + (base + c) * 8;
        lo[i] = __ldcg(reinterpret_cast<const float4*>(q));
        hi[i] = __ldcg(reinterpret_cast<const float4*>(q + 4));
      } else {
        pb[i] = reinterpret_cast<const uint4*>(partial)[base + c];
      }
    }
  }
  if (part) {
    for (int s = 1; s < S; ++s) {  // split order; the V chunks' loads of split s are independent
      float4 l2[V], h2[V];
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = c0 + threadIdx.x + i * kThreads;
        if (c < c1) {
          const float* q = part + s * plane + (base + c) * 8;
          l2[i] = __ldcg(reinterpret_cast<const float4*>(q));
          h2[i] = __ldcg(reinterpret_cast<const float4*>(q + 4));
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i) {
        add4(lo[i], l2[i]);
        add4(hi[i], h2[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&pb[i]);
      oh[0] = __floats2bfloat162_rn(lo[i].x, lo[i].y);
      oh[1] = __floats2bfloat162_rn(lo[i].z, lo[i].w);
      oh[2] = __floats2bfloat162_rn(hi[i].x, hi[i].y);
      oh[3] = __floats2bfloat162_rn(hi[i].z, hi[i].w);
    }
  }
  float f[V][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = c0 + threadIdx.x + i * kThreads;
    if (c < c1) {
      const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&xa[i]);
      const __nv_bfloat162* bh = reinterpret_cast<const __nv_bfloat162*>(&pb[i]);
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 u = __bfloat1622float2(ah[j]), v = __bfloat1622float2(bh[j]);
        oh[j] = __floats2bfloat162_rn(u.x + v.x, u.y + v.y);
        const float2 r = __bfloat1622float2(oh[j]);
        f[i][2 * j] = r.x;
        f[i][2 * j + 1] = r.y;
        ss += r.x * r.x + r.y * r.y;
      }
      xr[c] = o;
    }
  }
  const float t = block_sum(ss, red);
  float total = t;
  if (cpr > 1) {  // the cluster's CTA sums, in rank order, through distributed shared memory
    if (threadIdx.x == 0) cta_sum = t;
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    total = 0.f;
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(&cta_sum);
    for (int r = 0; r < cpr; ++r) {
      uint32_t remote;
      float v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
      total += v;
    }
    // peers may still read our cta_sum: stay resident until every CTA of the cluster has read
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  const float rstd = rsqrtf(total / (float)cols + eps);
  uint4* yr = reinterpret_cast<uint4*>(y) + base;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = c0 + threadIdx.x + i * kThreads;
    if (c < c1) {
      const __nv_bfloat162* wh = reinterpret_cast<const __nv_bfloat162*>(&wv[i]);
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 ww = __bfloat1622float2(wh[j]);
        oh[j] = __floats2bfloat162_rn(f[i][2 * j] * rstd * ww.x, f[i][2 * j + 1] * rstd * ww.y);
      }
      yr[c] = o;
    }
  }
  if (cpr > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  tstamp(tr, 3);
}

// launch: cpr = CTAs per row (a cluster), V = chunks per thread
static dak_status launch_residual_rmsnorm(const __nv_bfloat16* partial, const float* part, int S, void* x, int rows,
                                          int cols, const void* w, float eps, void* y, bool pdl, cudaStream_t s) {
  const int nc = cols / 8;
  const int cpr = std::min(kMaxCpr, std::max(1, (nc + kThreads - 1) / kThreads));
  const int per = (nc + cpr - 1) / cpr;
  const int V = (per + kThreads - 1) / kThreads;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cpr;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(rows * cpr);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  unsigned long long* tr = trace_slot(DAK_KIND_RESIDUAL, rows, cols, rows * cpr);
  auto go = [&](auto kern) {
    return cudaLaunchKernelEx(&cfg, kern, partial, (__nv_bfloat16*)x, cols, (const __nv_bfloat16*)w, eps,
                              (__nv_bfloat16*)y, part, S, rows, cpr, tr);
  };
  cudaError_t e;
  if (V <= 1) e = go(residual_rmsnorm_kernel<1>);
  else if (V <= 2) e = go(residual_rmsnorm_kernel<2>);
  else if (V <= 4) e = go(residual_rmsnorm_kernel<4>);
  else e = go(residual_rmsnorm_kernel<kVec>);
  DAK_CUDA_TRY(e);
  return DAK_OK;
}

// rank-major gather [world][N][Ml] -> row-major [N][world * Ml] (16-byte chunks; Ml % 8 == 0)
__global__ void gather_cols_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int world, int N, long long ml16) {
  const long long total = (long long)world * N * ml16;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i % ml16;
    const long long n = (i / ml16) % N;
    const long long r = i / (ml16 * N);
    dst[(n * world + r) * ml16 + c] = src[i];
  }
}

}  // namespace tp
}  // namespace dak

using namespace dak;

extern "C" {

dak_status dak_comm_unique_id(void* id_out) {
  if (!id_out) return fail(DAK_EINVAL, "dak_comm_unique_id: NULL");
  tp::Nccl* n;
  dak_status st = tp::nccl(&n);
  if (st != DAK_OK) return st;
  ncclUniqueId id;
  DAK_NCCL_TRY(n, n->get_unique_id(&id));
  memcpy(id_out, &id, sizeof(id));
  return DAK_OK;
}

dak_status dak_comm_init(const void* id, int32_t rank, int32_t world, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return fail(DAK_EINVAL, "dak_comm_init: bad arguments");
  tp::Nccl* n;
  dak_status st = tp::nccl(&n);
  if (st != DAK_OK) return st;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c;
  DAK_NCCL_TRY(n, n->comm_init_rank(&c, world, uid, rank));
  *comm = (void*)c;
  return DAK_OK;
}

dak_status dak_comm_destroy(void* comm) {
  if (!comm) return DAK_OK;
  tp::Nccl* n;
  dak_status st = tp::nccl(&n);
  if (st != DAK_OK) return st;
  DAK_NCCL_TRY(n, n->comm_destroy((ncclComm_t)comm));
  return DAK_OK;
}

dak_status dak_allreduce_residual(void* comm, void* partial, void* x, int32_t rows, int32_t cols, float* stats_out,
                                  int32_t pdl, dak_stream_t stream) {
  if (!partial || !x || rows <= 0 || cols <= 0) return fail(DAK_EINVAL, "dak_allreduce_residual: bad arguments");
  if (cols > tp::kThreads * tp::kPer) return fail(DAK_EUNSUPPORTED, "dak_allreduce_residual: cols > %d", tp::kThreads * tp::kPer);
  if (stats_out && !aligned16(stats_out)) return fail(DAK_EINVAL, "dak_allreduce_residual: stats_out must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (comm) {
    tp::Nccl* n;
    dak_status st = tp::nccl(&n);
    if (st != DAK_OK) return st;
    int world = 1;  // a one-rank communicator has nothing to exchange: no collective launch
    DAK_NCCL_TRY(n, n->comm_count((ncclComm_t)comm, &world));
    if (world > 1)
      DAK_NCCL_TRY(n, n->all_reduce(partial, partial, (size_t)rows * cols, ncclBfloat16, ncclSum, (ncclComm_t)comm, s));
    else
      comm = nullptr;  // PDL stays allowed below (no NCCL kernel in between)
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl && !comm) ? 1 : 0;  // NCCL kernels are not PDL-aware
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(rows);
  cfg.blockDim = dim3(tp::kThreads);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool vec = cols % 8 == 0 && cols <= tp::kThreads * 64 && aligned16(partial) && aligned16(x);
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, vec ? tp::residual_stats_vec_kernel : tp::residual_stats_kernel,
                                  (const __nv_bfloat16*)partial, (__nv_bfloat16*)x, (int)cols, (float4*)stats_out));
  return DAK_OK;
}

dak_status dak_comm_size(void* comm, int32_t* world) {
  if (!world) return fail(DAK_EINVAL, "dak_comm_size: NULL");
  if (!comm) {
    *world = 1;
    return DAK_OK;
  }
  tp::Nccl* n;
  dak_status st = tp::nccl(&n);
  if (st != DAK_OK) return st;
  int w = 0;
  DAK_NCCL_TRY(n, n->comm_count((ncclComm_t)comm, &w));
  *world = w;
  return DAK_OK;
}

dak_status dak_allgather_cols(void* comm, const void* send, void* recv, void* scratch, int32_t N, int64_t Ml,
                              dak_stream_t stream) {
  if (!send || !recv || N <= 0 || Ml <= 0) return fail(DAK_EINVAL, "dak_allgather_cols: bad arguments");
  if (Ml % 8 || !aligned16(send) || !aligned16(recv) || !aligned16(scratch))
    return fail(DAK_EINVAL, "dak_allgather_cols: Ml %% 8 == 0 and 16-byte aligned buffers required");
  int32_t world = 1;
  dak_status st = dak_comm_size(comm, &world);
  if (st != DAK_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t shard = (size_t)N * Ml;
  if (world == 1 || N == 1) {  // the rank-major gather already is row-major
    if (!comm) {
      if (recv != send) DAK_CUDA_TRY(cudaMemcpyAsync(recv, send, shard * 2, cudaMemcpyDeviceToDevice, s));
      return DAK_OK;
    }
    tp::Nccl* n;
    if ((st = tp::nccl(&n)) != DAK_OK) return st;
    DAK_NCCL_TRY(n, n->all_gather(send, recv, shard, ncclBfloat16, (ncclComm_t)comm, s));
    return DAK_OK;
  }
  if (!scratch) return fail(DAK_EINVAL, "dak_allgather_cols: scratch [world][N][Ml] needed for N > 1");
  tp::Nccl* n;
  if ((st = tp::nccl(&n)) != DAK_OK) return st;
  DAK_NCCL_TRY(n, n->all_gather(send, scratch, shard, ncclBfloat16, (ncclComm_t)comm, s));
  const long long ml16 = Ml / 8;
  const long long total = (long long)world * N * ml16;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  tp::gather_cols_kernel<<<grid, 256, 0, s>>>((const uint4*)scratch, (uint4*)recv, world, N, ml16);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

dak_status dak_allreduce_residual_rmsnorm(void* comm, void* partial, void* x, int32_t rows, int32_t cols,
                                          const void* norm_w, float eps, void* y_norm, int32_t pdl, dak_stream_t stream) {
  if (!partial || !x || !norm_w || !y_norm || rows <= 0 || cols <= 0)
    return fail(DAK_EINVAL, "dak_allreduce_residual_rmsnorm: bad arguments");
  if (cols % 8 || cols > tp::kThreads * 8 * tp::kVec * tp::kMaxCpr)
    return fail(DAK_EUNSUPPORTED, "dak_allreduce_residual_rmsnorm: cols must be a multiple of 8, <= %d",
                tp::kThreads * 8 * tp::kVec * tp::kMaxCpr);
  if (!aligned16(partial) || !aligned16(x) || !aligned16(norm_w) || !aligned16(y_norm))
    return fail(DAK_EINVAL, "dak_allreduce_residual_rmsnorm: pointers must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (comm) {
    tp::Nccl* n;
    dak_status st = tp::nccl(&n);
    if (st != DAK_OK) return st;
    int world = 1;  // a one-rank communicator has nothing to exchange: no collective launch
    DAK_NCCL_TRY(n, n->comm_count((ncclComm_t)comm, &world));
    if (world > 1)
      DAK_NCCL_TRY(n, n->all_reduce(partial, partial, (size_t)rows * cols, ncclBfloat16, ncclSum, (ncclComm_t)comm, s));
    else
      comm = nullptr;  // PDL stays allowed below (no NCCL kernel in between)
  }
  return tp::launch_residual_rmsnorm((const __nv_bfloat16*)partial, nullptr, 1, x, rows, cols, norm_w, eps, y_norm,
                                     pdl && !comm, s);  // NCCL kernels are not PDL-aware
}

}  // extern "C"

// One rank: x += bf16(sum_s part[s]) (split-K partials of the row-parallel linear, reduced here),
// y = RMSNorm(x) -- dak_allreduce_residual_rmsnorm with the reduce kernel folded in.
dak_status dak::residual_rmsnorm_part(const float* part, int32_t S, void* x, int32_t rows, int32_t cols,
                                      const void* norm_w, float eps, void* y_norm, int32_t pdl, void* stream) {
  if (!part || S < 1 || !x || !norm_w || !y_norm || rows <= 0 || cols <= 0 || cols % 8 ||
      cols > tp::kThreads * 8 * tp::kVec * tp::kMaxCpr || !aligned16(part) || !aligned16(x) || !aligned16(norm_w) ||
      !aligned16(y_norm))
    return fail(DAK_EINVAL, "residual_rmsnorm_part: bad arguments");
  return tp::launch_residual_rmsnorm(nullptr, part, S, x, rows, cols, norm_w, eps, y_norm, pdl != 0, (cudaStream_t)stream);
}
