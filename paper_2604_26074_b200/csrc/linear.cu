// dak_linear — split-source GEMV / skinny GEMM for sm_100a (PAPER §3.1).
//
//   y[n, m] = act( sum_k W[m, k] x[n, k] + bias[m] ) + residual[n, m]
//
// W is split along M: rows [0,h) live in pinned host memory reached over the
// CPU-GPU link, rows [h,M) in HBM. Each CTA reads exactly one tier: CTAs [0,n_host)
// own contiguous ranges of host rows, the rest contiguous ranges of HBM rows, sizes differing by
// at most one row (row-granular wave alignment). Inside a CTA one producer lane streams
// the CTA's rows chunk by chunk (KC columns at a time) into an SMEM ring with 1-D bulk copies
// (cp.async.bulk -> TMA engine, UBLKCP) completing on mbarriers; the same copy
// instruction serves both tiers because host memory is device-mapped (measured on the box:
// profiles/r01/calib_loadpath.jsonl). The number of host stages in flight is capped by the
// congestion window W. Consumer warps compute either on CUDA cores (N <= 4: FMA with a
// fixed per-thread k-slice, then warp-shuffle reduction) or on tensor cores (mma.sync
// m16n8k16 bf16 -> fp32) and a deterministic cross-warp reduction through SMEM.
//
// Weights use the DAK-KC layout (see include/dak.h): chunk-major [K/KC][rows][KC], 16-byte
// chunks of each 128-byte atom XOR-swizzled by (row & 7). One k-chunk of a contiguous row range
// is one contiguous span, so a pipeline stage is ONE bulk copy of W plus N small copies of x.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace dak {
namespace lin {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = 32 + kConsumers;  // warp 0 = producer
constexpr int kMaxN = 16;
constexpr int kRptMax = 16;   // FMA path: rows per thread
constexpr int kMtwMax = 12;   // MMA path: m16 tiles per warp
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 227 * 1024;

struct Params {
  const char* w_host;
  const char* w_hbm;
  long long M, K, h;
  int kc, N;
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int act;
  int n_host, n_hbm;
  int stages, window;
  int w_stage_bytes, x_stage_bytes, x_pitch;
  int res_offset;  // byte offset of the fp32 result buffer in smem
  long long ldy;   // elements between consecutive rows n of y and residual
};

// ------------------------------------------------------------------------------------ PTX glue
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// byte offset of 16-byte chunk `sl` of local row `r` inside a stage (row pitch = kc*2)
__device__ __forceinline__ uint32_t swz(long long r_tier, int sl) {
  return (uint32_t)(((sl >> 3) << 7) | (((sl & 7) ^ (int)(r_tier & 7)) << 4));
}

// ------------------------------------------------------------------------------------ kernel
// PATH 1: CUDA-core FMA, NN = N (1..4), MTW = rows per thread bucket.
// PATH 2: mma.sync,      NN = n8 tiles (1..2), MTW = m16 tiles per warp bucket.
// Every loop whose body holds a .sync.aligned instruction has a compile-time trip count, so the
// hot loop is branch-free (the first build spent ~30 SASS instructions per HMMA on predicates,
// WARPSYNC and ring-index divisions — profiles/r01/linear_v0_ncu.txt).
template <int PATH, int NN, int MTW>
__global__ void __launch_bounds__(kThreads, 1) split_linear_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* wring = smem + 1024;
  unsigned char* xring = wring + (size_t)p.stages * p.w_stage_bytes;
  float* res = reinterpret_cast<float*>(smem + p.res_offset);

  const int cta = blockIdx.x;
  const bool host = cta < p.n_host;
  long long rb, re;  // tier-local row range
  const long long R_tier = host ? p.h : p.M - p.h;
  {
    const long long j = host ? cta : cta - p.n_host;
    const long long n = host ? p.n_host : p.n_hbm;
    rb = j * R_tier / n;
    re = (j + 1) * R_tier / n;
  }
  const int R = (int)(re - rb);
  const long long row0 = host ? rb : p.h + rb;  // global row of local row 0
  const char* wsrc = host ? p.w_host : p.w_hbm;
  const int slots = host ? p.window : p.stages;
  const int kc = p.kc;
  const int nchunks = (int)(p.K / kc);
  const int N = p.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  grid_dep_launch();  // the next op may start its weight stream as our CTAs retire
  if (R <= 0) return;

  const uint32_t w_bytes = (uint32_t)R * kc * 2;
  const uint32_t x_bytes = (uint32_t)kc * 2;
  const long long chunk_stride = R_tier * kc * 2;  // bytes between consecutive k-chunks of a row

  if (warp == 0) {
    // ============================ producer: lane 0 streams W, lanes 0..N-1 stream x rows
    const int pro = min(slots, nchunks);
    const char* src = wsrc + rb * kc * 2;
    if (lane == 0) {
      for (int i = 0; i < pro; ++i) {  // weights do not depend on the previous kernel: start now
        mbar_expect_tx(&full[i], w_bytes + (uint32_t)N * x_bytes);
        bulk_g2s(wring + (size_t)i * p.w_stage_bytes, src + (long long)i * chunk_stride, w_bytes, &full[i]);
      }
    }
    grid_dep_wait();  // x is produced by the previous kernel
    __syncwarp();
    const __nv_bfloat16* xrow = p.x + (long long)lane * p.K;
    if (lane < N)
      for (int i = 0; i < pro; ++i)
        bulk_g2s(xring + (size_t)i * p.x_stage_bytes + lane * p.x_pitch, xrow + (long long)i * kc, x_bytes, &full[i]);
    int s = pro == slots ? 0 : pro;
    uint32_t ph = pro == slots ? 1u : 0u;
    for (int i = pro; i < nchunks; ++i) {
      if (lane == 0) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], w_bytes + (uint32_t)N * x_bytes);
        bulk_g2s(wring + (size_t)s * p.w_stage_bytes, src + (long long)i * chunk_stride, w_bytes, &full[s]);
      }
      __syncwarp();
      if (lane < N)
        bulk_g2s(xring + (size_t)s * p.x_stage_bytes + lane * p.x_pitch, xrow + (long long)i * kc, x_bytes, &full[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    return;
  }

  // ================================ consumers
  const int t = threadIdx.x - 32;
  const int cw = warp - 1;
  const uint32_t wring_u = su32(wring), xring_u = su32(xring);
  if constexpr (PATH == 1) {
    constexpr int RPT = MTW;
    const int S = kc >> 3;   // 16-byte slices per row chunk
    const int G = kConsumers / S;
    const int sl = t % S, rg = t / S;
    const uint32_t row_bytes = (uint32_t)kc * 2;
    // per-row byte offsets inside a stage (swizzle key = tier-local row & 7), hoisted out of the loop
    uint32_t roff[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int r = rg + G * j;
      roff[j] = (uint32_t)r * row_bytes + swz(rb + r, sl);
    }
    float acc[RPT][NN];
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int n = 0; n < NN; ++n) acc[j][n] = 0.f;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      const unsigned char* ws = wring + (size_t)s * p.w_stage_bytes;
      const unsigned char* xs = xring + (size_t)s * p.x_stage_bytes;
      float xf[NN][8];
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        const uint4 v = *reinterpret_cast<const uint4*>(xs + n * p.x_pitch + sl * 16);
        xf[n][0] = bf_lo(v.x); xf[n][1] = bf_hi(v.x); xf[n][2] = bf_lo(v.y); xf[n][3] = bf_hi(v.y);
        xf[n][4] = bf_lo(v.z); xf[n][5] = bf_hi(v.z); xf[n][6] = bf_lo(v.w); xf[n][7] = bf_hi(v.w);
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (rg + G * j < R) {
          const uint4 v = *reinterpret_cast<const uint4*>(ws + roff[j]);
          const float w[8] = {bf_lo(v.x), bf_hi(v.x), bf_lo(v.y), bf_hi(v.y), bf_lo(v.z), bf_hi(v.z), bf_lo(v.w), bf_hi(v.w)};
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            float a = acc[j][n];
#pragma unroll
            for (int e = 0; e < 8; ++e) a = fmaf(w[e], xf[n][e], a);
            acc[j][n] = a;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    // reduce the S slice-partials of each row: shuffle inside groups of min(S,32) lanes ...
    const int L = S < 32 ? S : 32;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int n = 0; n < NN; ++n)
        for (int off = L >> 1; off >= 1; off >>= 1) acc[j][n] += __shfl_xor_sync(0xffffffffu, acc[j][n], off);
    // ... then across the S/32 warps of a row group in fixed order through SMEM
    const int W2 = S > 32 ? S / 32 : 1;
    const int wg = (t % S) >> 5;
    if ((t % L) == 0) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int r = rg + G * j;
        if (r < R)
#pragma unroll
          for (int n = 0; n < NN; ++n) res[((size_t)wg * R + r) * NN + n] = acc[j][n];
      }
    }
    consumer_sync();
    if (W2 > 1) {
      for (int q = t; q < R * NN; q += kConsumers) {
        float a = res[q];
        for (int w2 = 1; w2 < W2; ++w2) a += res[(size_t)w2 * R * NN + q];
        res[q] = a;  // each q read+written by one thread; slots w2>=1 untouched
      }
      consumer_sync();
    }
  } else {
    constexpr int NT = NN;  // n8 tiles
    const int KS = kc >> 4;
    const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
    const int WM = kConsumerWarps / WK;
    const int wk = cw % WK, wm = cw / WK;
    const int nks = KS / WK;  // k-steps per warp per stage
    const int MT = (R + 15) >> 4;
    float acc[MTW][NT][4];
#pragma unroll
    for (int a = 0; a < MTW; ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
    const uint32_t row_bytes = (uint32_t)kc * 2;
    // A rows: tile mt = wm + WM*mi covers rows 16*mt .. +15; lane supplies row (lane & 15).
    // All tiles of a warp are 16*WM rows apart, so the swizzle key (row & 7) is per-thread constant.
    const uint32_t a_base = (uint32_t)(wm * 16 + (lane & 15)) * row_bytes;
    const uint32_t a_step = (uint32_t)(WM * 16) * row_bytes;
    const int key = (int)((rb + wm * 16 + (lane & 15)) & 7);
    const int ahalf = lane >> 4;
    const uint32_t b_base = (uint32_t)((lane & 7) + ((lane >> 4) << 3)) * p.x_pitch + ((lane >> 3) & 1) * 16;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      const uint32_t ws = wring_u + (uint32_t)s * p.w_stage_bytes + a_base;
      const uint32_t xs = xring_u + (uint32_t)s * p.x_stage_bytes + b_base;
      for (int j = 0; j < nks; ++j) {
        const int ks = wk + j * WK;
        uint32_t b[NT][2];
        if constexpr (NT == 1) {
          ldsm_x2(xs + ks * 32, b[0][0], b[0][1]);
        } else {
          ldsm_x4(xs + ks * 32, b[0][0], b[0][1], b[1][0], b[1][1]);
        }
        const int sl = 2 * ks + ahalf;
        const uint32_t coff = (uint32_t)(((sl >> 3) << 7) | (((sl & 7) ^ key) << 4));
#pragma unroll
        for (int mi = 0; mi < MTW; ++mi) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4(ws + mi * a_step + coff, a0, a1, a2, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_bf16(acc[mi][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    // deterministic cross-warp reduction over the WK warps sharing m-tiles (fixed wk order)
    const int g = lane >> 2, c2 = (lane & 3) * 2;
    for (int round = 0; round < WK; ++round) {
      if (wk == round) {
#pragma unroll
        for (int mi = 0; mi < MTW; ++mi) {
          const int mt = wm + WM * mi;
          if (mt < MT) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int r = mt * 16 + g + (c >> 1) * 8;
                const int n = nt * 8 + c2 + (c & 1);
                if (r < R && n < N) {
                  float* q = &res[(size_t)r * N + n];
                  *q = round == 0 ? acc[mi][nt][c] : *q + acc[mi][nt][c];
                }
              }
          }
        }
      }
      consumer_sync();
    }
  }

  // ================================ epilogue: bias, activation, residual, bf16 RNE store
  grid_dep_wait();  // residual / y may belong to the previous kernel
  const int RN = PATH == 1 ? NN : N;
  for (int q = t; q < R * N; q += kConsumers) {
    const int n = q / R, r = q - n * R;
    float v = res[(size_t)r * RN + n];
    const long long m = row0 + r;
    if (p.bias) v += __bfloat162float(p.bias[m]);
    if (p.act == DAK_ACT_RELU) v = fmaxf(v, 0.f);
    if (p.residual) v += __bfloat162float(p.residual[(long long)n * p.ldy + m]);
    p.y[(long long)n * p.ldy + m] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------------------------ packing
// dst[c][r][kc] with 16-byte chunk sl of row r stored at swz(r, sl); one thread per 16 B.
__global__ void pack_kernel(const uint4* __restrict__ src, long long rows, long long K, int kc, uint4* __restrict__ dst) {
  const long long per_row = K / 8;
  const long long total = rows * per_row;
  const int S = kc / 8;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / per_row;
    const long long q = idx % per_row;  // 16-byte chunk index along K
    const long long c = q / S;
    const int sl = (int)(q % S);
    const long long base = (c * rows + r) * (long long)kc * 2;  // bytes
    const uint32_t off = (uint32_t)(((sl >> 3) << 7) | (((sl & 7) ^ (int)(r & 7)) << 4));
    dst[(base + off) / 16] = src[idx];
  }
}

// ------------------------------------------------------------------------------------ host side
struct Plan {
  Params p;
  int path, nn, bucket, grid, smem;
  long long rmax_host, rmax_hbm;
};

static int g_sms = 0;
static dak_status device_sms(int* out) {
  if (g_sms <= 0) {
    int dev = 0;
    DAK_CUDA_TRY(cudaGetDevice(&dev));
    DAK_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  *out = g_sms;
  return DAK_OK;
}

static inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// compiled unroll buckets: FMA rows-per-thread and MMA m16-tiles-per-warp
static const int kRptBuckets[] = {1, 2, 4, 8, 16};
static const int kMtwBuckets[] = {1, 2, 3, 4, 6, 8, 12};

static int bucket_of(const int* b, int n, long long need) {
  for (int i = 0; i < n; ++i)
    if (b[i] >= need) return b[i];
  return -1;
}

// Rows a CTA may own for a given KC (accumulator capacity of each path).
static long long path_row_cap(int path, int kc) {
  if (path == 1) {
    const int S = kc / 8;
    return (long long)(kConsumers / S) * kRptMax;
  }
  const int KS = kc / 16;
  const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
  return 16LL * (kConsumerWarps / WK) * kMtwMax;
}

static dak_status make_plan(const dak_linear_args* a, Plan* out) {
  if (!a) return fail(DAK_EINVAL, "dak_linear: args NULL");
  const long long M = a->M, K = a->K, h = a->h;
  const int N = a->N, kc = a->kc;
  if (M <= 0 || K <= 0 || N <= 0) return fail(DAK_EINVAL, "dak_linear: M, K, N must be positive");
  if (h < 0 || h > M) return fail(DAK_EINVAL, "dak_linear: h must be in [0, M]");
  if (N > kMaxN) return fail(DAK_EUNSUPPORTED, "dak_linear: N=%d > %d (tcgen05 large-N path not in this build)", N, kMaxN);
  if (K % 64) return fail(DAK_EUNSUPPORTED, "dak_linear: K %% 64 != 0");
  if (kc < 64 || kc > 2048 || (kc & (kc - 1)) || K % kc)
    return fail(DAK_EINVAL, "dak_linear: kc must be a power of two in [64, 2048] dividing K");
  if (!a->x || !a->y) return fail(DAK_EINVAL, "dak_linear: x/y NULL");
  if ((h > 0 && !a->w_host) || (h < M && !a->w_hbm)) return fail(DAK_EINVAL, "dak_linear: missing weight tier pointer");
  if (!aligned16(a->x) || !aligned16(a->w_host) || !aligned16(a->w_hbm))
    return fail(DAK_EINVAL, "dak_linear: x and weight pointers must be 16-byte aligned");
  if (a->act != DAK_ACT_NONE && a->act != DAK_ACT_RELU) return fail(DAK_EINVAL, "dak_linear: bad act");

  const dak_launch_cfg& c = a->cfg;
  int sms = 0;
  if (h < M && c.n_cta_hbm <= 0) {  // auto sizing needs the device; explicit sizes are pure
    dak_status st = device_sms(&sms);
    if (st != DAK_OK) return st;
  }
  // default: tensor-core path for every N (the CUDA-core FMA loop cannot issue fast enough to
  // keep up with HBM); force_path 1 selects it for N <= 4.
  int path = c.force_path ? c.force_path : 2;
  if (path == 1 && N > 4) return fail(DAK_EUNSUPPORTED, "dak_linear: CUDA-core path supports N <= 4");
  if (path != 1 && path != 2) return fail(DAK_EINVAL, "dak_linear: bad force_path");
  // rows per CTA are bounded by the accumulator capacity of the path and by SMEM: at least three
  // ring stages of (rows x KC) weights plus the x rows must fit (deep enough to cover HBM latency)
  const long long x_stage = ceil_div((long long)ceil_div(N, 8) * 8 * (kc * 2 + 16), 128) * 128;
  const long long smem_rows = ((kSmemBudget - 1024 - 8192) / 3 - x_stage) / (kc * 2) / 16 * 16;
  const long long cap = std::min(path_row_cap(path, kc), smem_rows);
  if (cap < 16) return fail(DAK_EUNSUPPORTED, "dak_linear: kc=%d leaves no room for a 16-row stage", kc);

  int n_host = 0;
  if (h > 0) {
    n_host = c.n_cta_host > 0 ? c.n_cta_host : 1;
    n_host = (int)std::max<long long>(n_host, ceil_div(h, cap));
    n_host = (int)std::min<long long>(n_host, h);
  }
  int n_hbm = 0;
  if (h < M) {
    n_hbm = c.n_cta_hbm > 0 ? c.n_cta_hbm : std::max(1, sms - n_host);
    n_hbm = (int)std::max<long long>(n_hbm, ceil_div(M - h, cap));
    n_hbm = (int)std::min<long long>(n_hbm, M - h);
  }
  const long long rmax_host = n_host ? ceil_div(h, n_host) : 0;
  const long long rmax_hbm = n_hbm ? ceil_div(M - h, n_hbm) : 0;
  const long long rmax = std::max(rmax_host, rmax_hbm);
  if (rmax > cap) return fail(DAK_EUNSUPPORTED, "dak_linear: %lld rows per CTA exceed the path capacity %lld (use a smaller kc)", rmax, cap);

  // unroll bucket and the rows one stage must hold (MMA tiles read whole 16-row groups)
  long long rows_alloc;
  int bucket;
  if (path == 1) {
    const int G = kConsumers / (kc / 8);
    bucket = bucket_of(kRptBuckets, 5, ceil_div(rmax, G));
    rows_alloc = ceil_div(rmax, 16) * 16;
  } else {
    const int KS = kc / 16;
    const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
    const int WM = kConsumerWarps / WK;
    bucket = bucket_of(kMtwBuckets, 7, ceil_div(ceil_div(rmax, 16), WM));
    rows_alloc = (long long)WM * bucket * 16;
  }
  if (bucket < 0) return fail(DAK_EUNSUPPORTED, "dak_linear: no unroll bucket for %lld rows per CTA", rmax);

  Params p{};
  p.w_host = (const char*)a->w_host;
  p.w_hbm = (const char*)a->w_hbm;
  p.M = M; p.K = K; p.h = h; p.kc = kc; p.N = N;
  p.x = (const __nv_bfloat16*)a->x;
  p.y = (__nv_bfloat16*)a->y;
  p.bias = (const __nv_bfloat16*)a->bias;
  p.residual = (const __nv_bfloat16*)a->residual;
  p.act = a->act;
  p.ldy = a->ldy > 0 ? a->ldy : M;
  if (p.ldy < M) return fail(DAK_EINVAL, "dak_linear: ldy < M");
  p.n_host = n_host; p.n_hbm = n_hbm;
  p.w_stage_bytes = (int)(rows_alloc * kc * 2);
  p.x_pitch = kc * 2 + 16;
  const int x_rows = path == 1 ? N : (int)ceil_div(N, 8) * 8;
  p.x_stage_bytes = (int)(ceil_div((long long)x_rows * p.x_pitch, 128) * 128);
  const int W2 = (path == 1 && kc / 8 > 32) ? kc / 8 / 32 : 1;
  const int res_bytes = (int)(ceil_div((long long)W2 * rmax * N * 4, 128) * 128);
  const int per_stage = p.w_stage_bytes + p.x_stage_bytes;
  int max_stages = (kSmemBudget - 1024 - res_bytes) / per_stage;
  if (max_stages < 2) return fail(DAK_EUNSUPPORTED, "dak_linear: stage of %d B does not fit twice in SMEM (use a smaller kc)", per_stage);
  max_stages = std::min(max_stages, kMaxStages);
  int stages = c.stages > 0 ? std::min(c.stages, max_stages) : max_stages;
  if (stages < 2) stages = 2;
  p.stages = stages;
  // congestion window: in-flight host stages per host CTA. With congestion control the
  // window is the smallest that keeps ~192 KB in flight on the link (calibrated saturation point,
  // profiles/r01/calib_loadpath.jsonl); without it every ring slot may be in flight.
  int window = stages;
  if (n_host > 0) {
    if (c.window > 0) window = std::min(c.window, stages);
    else if (c.congestion_control) {
      const long long hstage = std::max<long long>(1, rmax_host * kc * 2);
      window = (int)std::min<long long>(stages, std::max<long long>(1, ceil_div(192 * 1024, hstage * n_host)));
    }
  }
  p.window = std::max(1, window);
  p.res_offset = 1024 + stages * per_stage;

  out->p = p;
  out->path = path;
  out->nn = path == 1 ? N : (int)ceil_div(N, 8);
  out->bucket = bucket;
  out->grid = n_host + n_hbm;
  out->smem = p.res_offset + res_bytes;
  out->rmax_host = rmax_host;
  out->rmax_hbm = rmax_hbm;
  return DAK_OK;
}

template <int PATH, int NN, int B>
static dak_status launch_t(const Plan& pl, cudaStream_t stream, int pdl) {
  auto kern = split_linear_kernel<PATH, NN, B>;
  static int smem_set = 0;  // raise the opt-in limit once per instance (not a stream op; capture-safe)
  if (!smem_set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    smem_set = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, pl.p));
  return DAK_OK;
}

template <int PATH, int NN>
static dak_status launch_b(const Plan& pl, cudaStream_t s, int pdl) {
  if constexpr (PATH == 1) {
    switch (pl.bucket) {
      case 1: return launch_t<1, NN, 1>(pl, s, pdl);
      case 2: return launch_t<1, NN, 2>(pl, s, pdl);
      case 4: return launch_t<1, NN, 4>(pl, s, pdl);
      case 8: return launch_t<1, NN, 8>(pl, s, pdl);
      case 16: return launch_t<1, NN, 16>(pl, s, pdl);
    }
  } else {
    switch (pl.bucket) {
      case 1: return launch_t<2, NN, 1>(pl, s, pdl);
      case 2: return launch_t<2, NN, 2>(pl, s, pdl);
      case 3: return launch_t<2, NN, 3>(pl, s, pdl);
      case 4: return launch_t<2, NN, 4>(pl, s, pdl);
      case 6: return launch_t<2, NN, 6>(pl, s, pdl);
      case 8: return launch_t<2, NN, 8>(pl, s, pdl);
      case 12: return launch_t<2, NN, 12>(pl, s, pdl);
    }
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no kernel instance for bucket %d", pl.bucket);
}

static dak_status launch(const Plan& pl, cudaStream_t s, int pdl) {
  if (pl.grid == 0) return DAK_OK;
  if (pl.path == 1) {
    switch (pl.nn) {
      case 1: return launch_b<1, 1>(pl, s, pdl);
      case 2: return launch_b<1, 2>(pl, s, pdl);
      case 3: return launch_b<1, 3>(pl, s, pdl);
      case 4: return launch_b<1, 4>(pl, s, pdl);
    }
  } else {
    switch (pl.nn) {
      case 1: return launch_b<2, 1>(pl, s, pdl);
      case 2: return launch_b<2, 2>(pl, s, pdl);
    }
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no kernel instance for path %d / %d", pl.path, pl.nn);
}

}  // namespace lin
}  // namespace dak

using namespace dak;

extern "C" {

size_t dak_linear_packed_bytes(int64_t rows, int64_t K, int32_t kc) {
  (void)kc;
  return (size_t)rows * (size_t)K * 2;
}

int32_t dak_linear_default_kc(int64_t M, int64_t K, int32_t n_ctas) {
  // largest power-of-two KC (64..1024) dividing K with rows_per_cta * KC * 2 <= 40 KB
  if (n_ctas <= 0) n_ctas = 148;
  const long long r = (M + n_ctas - 1) / n_ctas;
  int best = 64;
  for (int kc = 64; kc <= 1024; kc *= 2) {
    if (K % kc) break;
    if (r * kc * 2 <= 40 * 1024) best = kc;
  }
  return best;
}

dak_status dak_pack_linear(const void* src, int64_t rows, int64_t K, int32_t kc, void* dst, dak_stream_t stream) {
  if (!src || !dst || rows < 0 || K <= 0) return fail(DAK_EINVAL, "dak_pack_linear: bad arguments");
  if (K % 64 || kc < 64 || kc > 2048 || (kc & (kc - 1)) || K % kc)
    return fail(DAK_EINVAL, "dak_pack_linear: need K %% 64 == 0 and power-of-two kc in [64,2048] dividing K");
  if (!aligned16(src) || !aligned16(dst)) return fail(DAK_EINVAL, "dak_pack_linear: pointers must be 16-byte aligned");
  if (rows == 0) return DAK_OK;
  const long long total = rows * (K / 8);
  const int threads = 256;
  const long long blocks = std::min<long long>((total + threads - 1) / threads, 148LL * 64);
  lin::pack_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, rows, K, kc, (uint4*)dst);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

dak_status dak_linear_query(const dak_linear_args* args, dak_linear_launch_info* info) {
  if (!info) return fail(DAK_EINVAL, "dak_linear_query: info NULL");
  lin::Plan pl;
  dak_status st = lin::make_plan(args, &pl);
  if (st != DAK_OK) return st;
  info->grid = pl.grid;
  info->n_cta_host = pl.p.n_host;
  info->n_cta_hbm = pl.p.n_hbm;
  info->threads = lin::kThreads;
  info->stages_hbm = pl.p.stages;
  info->window_host = pl.p.window;
  info->smem_bytes = pl.smem;
  info->path = pl.path;
  info->rows_per_cta_host_max = pl.rmax_host;
  info->rows_per_cta_hbm_max = pl.rmax_hbm;
  info->hbm_bytes = (args->M - args->h) * args->K * 2;
  info->host_bytes = args->h * args->K * 2;
  return DAK_OK;
}

dak_status dak_linear_cta_rows(const dak_linear_args* args, int32_t cta, int32_t* tier, int64_t* row_begin, int64_t* row_end) {
  if (!tier || !row_begin || !row_end) return fail(DAK_EINVAL, "dak_linear_cta_rows: NULL output");
  lin::Plan pl;
  dak_status st = lin::make_plan(args, &pl);
  if (st != DAK_OK) return st;
  if (cta < 0 || cta >= pl.grid) return fail(DAK_EINVAL, "dak_linear_cta_rows: cta out of range");
  const bool host = cta < pl.p.n_host;
  const long long R = host ? args->h : args->M - args->h;
  const long long j = host ? cta : cta - pl.p.n_host;
  const long long n = host ? pl.p.n_host : pl.p.n_hbm;
  const long long off = host ? 0 : args->h;
  *tier = host ? 1 : 0;
  *row_begin = off + j * R / n;
  *row_end = off + (j + 1) * R / n;
  return DAK_OK;
}

dak_status dak_linear(const dak_linear_args* args, dak_stream_t stream) {
  lin::Plan pl;
  dak_status st = lin::make_plan(args, &pl);
  if (st != DAK_OK) return st;
  if (pl.grid && !(pl.p.y)) return fail(DAK_EINVAL, "dak_linear: y NULL");
  return lin::launch(pl, (cudaStream_t)stream, args->cfg.pdl);
}

}  // extern "C"
