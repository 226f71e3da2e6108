// dak_linear_chain -- a chain of split GEMVs (§3.1, the dak_linear operator) run by ONE
// persistent grid: one CTA per SM walks the ops in order, and its producer lane streams the weights
// of op i+1 (HBM rows, or host rows under the congestion window) into the same SMEM ring
// while the consumer warps still compute op i. Between launches of dak_linear every SM drains its
// ring, exits and restarts the next op's ring from empty (~2-3 us per op: the C1 4096^2 GEMV takes
// 7.3 us per chained launch against ~4.6 us of streaming); here the ring never drains.
//
// Dependencies: op i whose x / residual / y overlap an earlier op's buffers (a decode chain: x of op
// i is y of op i-1) waits until every CTA has finished op i-1 -- a per-op counter of CTAs done in
// the workspace (release: fence + atomicAdd; acquire + proxy fence before the x tensor TMA). Only
// the x loads (and so the MMAs) wait: weight stages of later ops are already in flight. The grid is
// one CTA per SM (all co-resident), so the counter waits cannot deadlock.
//
// Per op and CTA the arithmetic is dak_linear's mma.sync path (the same row partition, the same
// k-step split across warps, the same fixed-order cross-warp reduction and epilogue): every output
// is bitwise equal to the op launched alone with the same kc (tested).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "ptx.cuh"

namespace dak {
namespace chain {

using namespace ptx;

constexpr int kMaxOps = 16;
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = 32 + kConsumers + 64;  // W producer, 8 consumer warps, x producer, signal warp
constexpr int kMaxStages = 16;
constexpr int kSmemBudget = 227 * 1024;

struct __align__(64) Op {
  CUtensorMap xmap;  // x [N, K] as (64 elements, N rows, K/64 atoms), 128-byte swizzle (dak_linear's)
  const char* w_host;
  const char* w_hbm;
  long long M, K, h, ldy;
  __nv_bfloat16* y;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int act, n_host, n_hbm, window;  // window: in-flight host stages per host CTA
  int dep;                         // 1: wait for every CTA to finish op - 1 before reading x / residual
  int nchunks;                     // K / kc
};

struct __align__(64) Params {
  Op ops[kMaxOps];
  int n_ops, kc, N, n8, stages, w_stage_bytes, x_stage_bytes, off_x, res_offset, wm, wk, red_slots;
  int xres_bytes;  // x-resident mode: bytes of one of the two whole-x buffers (0: an x box per stage)
  int evict_first;
  int* done;  // [n_ops] CTAs that finished op i (workspace; the last CTA of the chain zeroes it again)
  unsigned long long* trace;
};

__device__ __forceinline__ void tier_rows(long long R, long long j, long long n, long long* rb, long long* re) {
  const long long b = j * R / n, e = (j + 1) * R / n;  // sizes differ by <= 1 row (dak_linear's rgran 1)
  *rb = b;
  *re = e;
}
__device__ __forceinline__ void op_rows(const Op& o, int cta, bool* host, long long* rb, long long* re, long long* R_tier) {
  *host = cta < o.n_host;
  *R_tier = *host ? o.h : o.M - o.h;
  const long long j = *host ? cta : cta - o.n_host;
  const long long n = *host ? o.n_host : o.n_hbm;
  if (n <= 0 || j >= n) {
    *rb = *re = 0;
    return;
  }
  tier_rows(*R_tier, j, n, rb, re);
}
__device__ __forceinline__ void bulk_g2s_ef(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && blockIdx.x < kTraceCtas) tr[blockIdx.x * 4 + k] = gtime();
}
// EXPERIMENT: per-op stamps in the launch trace, virtual CTA = cta + grid * op (ops * grid <= 1024)
__device__ __forceinline__ void ostamp(unsigned long long* tr, int op, int k) {
  const unsigned v = blockIdx.x + gridDim.x * op;
  if (tr && v < (unsigned)kTraceCtas) tr[v * 4 + k] = gtime();
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

// XRES (x-resident): every op's whole x [N, K] is one tensor box loaded once per op into one of two
// SMEM buffers (ping-pong, xfull / xempty barriers), so a ring stage is weights only and the ring
// holds most of an op's weights while its dependency resolves. Else an x box per stage.
template <int NT, int MTW, bool XRES>
__global__ void __launch_bounds__(kThreads, 1) chain_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* wring = smem + 1024;
  unsigned char* xring = smem + p.off_x;
  float* res = reinterpret_cast<float*>(smem + p.res_offset);
  const int cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc = p.kc, N = p.N, stages = p.stages;
  const int grid = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    *reinterpret_cast<volatile int*>(full + 2 * kMaxStages) = 0;
    for (int b = 0; b < 2; ++b) {
      mbar_init(full + 2 * kMaxStages + 1 + b, 1);
      mbar_init(full + 2 * kMaxStages + 3 + b, kConsumerWarps);
    }
    for (int i = 0; i < kMaxOps; ++i) mbar_init(full + 2 * kMaxStages + 5 + i, kConsumerWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  volatile int* w_issued = reinterpret_cast<volatile int*>(empty + kMaxStages);  // W stages whose expect_tx is set
  uint64_t* xfull = empty + kMaxStages + 1;  // [2] x buffer b holds the x of the current op using it
  uint64_t* xempty = xfull + 2;              // [2] the consumers are done with x buffer b
  uint64_t* epi = xempty + 2;                // [kMaxOps] the consumers stored this CTA's y slice of op i
  if (warp == 0) {
    // ============================ W producer: weight stages run ahead across ops (ring-bounded)
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      long long g = 0;
      for (int oi = 0; oi < p.n_ops; ++oi) {
        const Op& o = p.ops[oi];
        bool h_;
        long long rb, re, Rt;
        op_rows(o, cta, &h_, &rb, &re, &Rt);
        if (re <= rb) continue;  // no rows of this op here
        const uint32_t wb = (uint32_t)((re - rb) * kc * 2);
        const char* src = (h_ ? o.w_host : o.w_hbm) + rb * kc * 2;
        const long long cstride = Rt * kc * 2;
        for (int c = 0; c < o.nchunks; ++c, ++g) {
          const int s = (int)(g % stages);
          if (g >= stages) mbar_wait(&empty[s], (uint32_t)(((g / stages) - 1) & 1));
          if (h_ && o.window < stages && g >= o.window) {  // congestion window: <= window host stages in flight
            const long long g0 = g - o.window;
            mbar_wait(&full[g0 % stages], (uint32_t)((g0 / stages) & 1));
          }
          mbar_expect_tx(&full[s], wb + (XRES ? 0u : (uint32_t)p.x_stage_bytes));
          if (p.evict_first) bulk_g2s_ef(wring + (size_t)s * p.w_stage_bytes, src + c * cstride, wb, &full[s], pol);
          else bulk_g2s(wring + (size_t)s * p.w_stage_bytes, src + c * cstride, wb, &full[s]);
          __threadfence_block();
          *w_issued = (int)(g + 1);
        }
      }
    }
    return;
  }
  if (warp == kConsumerWarps + 1) {
    // ============================ x producer: each stage's x box once its W stage is armed and its
    // op's dependency is met (the previous kernel for the first ops; every CTA done with op - 1 for
    // a dependent op)
    if (lane == 0) {
      for (int i = 0; i < p.n_ops; ++i)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.ops[i].xmap)) : "memory");
      // x of the first ops comes from the previous kernel, and the counters of this launch are
      // zero only once the previous launch (whose CTA 0 zeroes them) has completed: wait first
      asm volatile("griddepcontrol.wait;" ::: "memory");
      long long g = 0;
      int xi = 0;  // XRES: ops (with rows here) whose x has been loaded
      for (int oi = 0; oi < p.n_ops; ++oi) {
        const Op& o = p.ops[oi];
        bool h_;
        long long rb, re, Rt;
        op_rows(o, cta, &h_, &rb, &re, &Rt);
        if (re <= rb) continue;
        if (oi > 0 && o.dep) {
          // acquire polls (one L2 round trip per check); bounded: a CTA that never arrives is a bug
          // and traps (a kernel error) instead of hanging the device
          for (long long it = 0; ld_acquire(p.done + (oi - 1)) < grid; ++it)
            if (it > (1LL << 26)) asm volatile("trap;");
          fence_proxy_async();  // other CTAs' generic y stores -> this CTA's async-proxy x loads
        }
        ostamp(p.trace, oi, 1);
        if constexpr (XRES) {  // the op's whole x into buffer xi & 1, once its previous user is done
          const int b = xi & 1;
          if (xi >= 2) mbar_wait(&xempty[b], (uint32_t)(((xi >> 1) - 1) & 1));
          mbar_expect_tx(&xfull[b], (uint32_t)(p.N * o.K * 2));
          tma_3d(xring + (size_t)b * p.xres_bytes, reinterpret_cast<uint64_t>(&o.xmap), 0, 0, 0, &xfull[b]);
          ++xi;
        } else {
          for (int c = 0; c < o.nchunks; ++c, ++g) {
            while (*w_issued <= g) __nanosleep(20);
            const int s = (int)(g % stages);
            tma_3d(xring + (size_t)s * p.x_stage_bytes, reinterpret_cast<uint64_t>(&o.xmap), 0, 0, c * (kc >> 6), &full[s]);
          }
        }
      }
    }
    return;
  }

  if (warp == kConsumerWarps + 2) {
    // ============================ signal warp: publishes "this CTA is done with op i" (release at
    // gpu scope, cumulative over the consumers' y stores observed through epi[i]), off the
    // consumers' path so they move on to the next op at once
    if (lane == 0) {
      for (int oi = 0; oi < p.n_ops; ++oi) {
        bool h_;
        long long rb, re, Rt;
        op_rows(p.ops[oi], cta, &h_, &rb, &re, &Rt);
        if (re > rb) mbar_wait(&epi[oi], 0);
        red_release_add(p.done + oi, 1);
        ostamp(p.trace, oi, 3);
      }
      if (cta == 0) {
        // every CTA passed every wait once all have finished the last op: zero the counters for
        // the next call (CTA 0 waits for the others here, at the very end of the chain)
        const int last = p.n_ops - 1;
        for (long long it = 0; ld_acquire(p.done + last) < grid; ++it) {
          __nanosleep(64);
          if (it > (1LL << 24)) asm volatile("trap;");
        }
        for (int i = 0; i < p.n_ops; ++i) p.done[i] = 0;
        __threadfence();
      }
    }
    return;
  }

  // ================================ consumers: dak_linear's mma.sync path, op after op
  const int t = threadIdx.x - 32;
  const int cw = warp - 1;
  const int KS = kc >> 4;
  const int WK = p.wk, WM = p.wm;
  const int wk = cw % WK, wm = cw / WK;
  const int nks = KS / WK;
  const uint32_t row_bytes = (uint32_t)kc * 2;
  const uint32_t a_base = (uint32_t)(wm * 16 + (lane & 15)) * row_bytes;
  const uint32_t a_step = (uint32_t)(WM * 16) * row_bytes;
  const int ahalf = lane >> 4;
  const int bn = (lane & 7) + ((lane >> 4) << 3);
  const int bjh = (lane >> 3) & 1;
  const uint32_t b_row = (uint32_t)bn << 7;
  const uint32_t atom_bytes = (uint32_t)p.n8 << 7;
  const uint32_t wring_u = su32(wring), xring_u = su32(xring);
  const int g8 = lane >> 2, c2 = (lane & 3) * 2;
  long long gs = 0;  // global stage index (matches the producer's)
  int xc = 0;        // XRES: ops with rows here consumed so far (x buffer xc & 1)
  for (int oi = 0; oi < p.n_ops; ++oi) {
    const Op& o = p.ops[oi];
    bool host;
    long long rb, re, Rt;
    op_rows(o, cta, &host, &rb, &re, &Rt);
    const int R = (int)(re - rb);
    const long long row0 = host ? rb : o.h + rb;
    if (R > 0) {
      const int MT = (R + 15) >> 4;
      const int key = (int)((rb + wm * 16 + (lane & 15)) & 7);
      float acc[MTW][NT][4];
#pragma unroll
      for (int a = 0; a < MTW; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
      const int xb = xc & 1;
      if constexpr (XRES) mbar_wait(&xfull[xb], (uint32_t)((xc >> 1) & 1));
      for (int i = 0; i < o.nchunks; ++i, ++gs) {
        const int s = (int)(gs % stages);
        mbar_wait(&full[s], (uint32_t)((gs / stages) & 1));
        if (i == 0 && t == 0) ostamp(p.trace, oi, 0);
        const uint32_t ws = wring_u + (uint32_t)s * p.w_stage_bytes + a_base;
        const uint32_t xs = XRES ? xring_u + (uint32_t)xb * p.xres_bytes : xring_u + (uint32_t)s * p.x_stage_bytes + b_row;
        for (int j = 0; j < nks; ++j) {
          const int ks = wk + j * WK;
          uint32_t b[NT][2];
          const int c8 = ((ks & 3) << 1) + bjh;
          uint32_t baddr;
          if constexpr (XRES) {  // line L = atom * N + row of the whole-x box (128B swizzle: chunk ^ (L & 7))
            const int L = (i * (kc >> 6) + (ks >> 2)) * N + bn;
            baddr = xs + (uint32_t)(L << 7) + (uint32_t)((c8 ^ (L & 7)) << 4);
          } else {
            baddr = xs + (uint32_t)(ks >> 2) * atom_bytes + (uint32_t)((c8 ^ (bn & 7)) << 4);
          }
          if constexpr (NT == 1) {
            ldsm_x2(baddr, b[0][0], b[0][1]);
          } else {
            ldsm_x4(baddr, b[0][0], b[0][1], b[1][0], b[1][1]);
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
      }
      if constexpr (XRES) {  // x buffer xb is free for the op after next
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[xb]);
        ++xc;
      }
      if (t == 0) ostamp(p.trace, oi, 2);
      // fixed-order cross-warp reduction over the WK warps sharing m-tiles (dak_linear's)
      if (p.red_slots > 1) {
        float* slot = res + (size_t)wk * R * N;
#pragma unroll
        for (int mi = 0; mi < MTW; ++mi) {
          const int mt = wm + WM * mi;
          if (mt < MT) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int r = mt * 16 + g8 + (c >> 1) * 8;
                const int n = nt * 8 + c2 + (c & 1);
                if (r < R && n < N) slot[(size_t)r * N + n] = acc[mi][nt][c];
              }
          }
        }
      }
      for (int round = 0; round < (p.red_slots > 1 ? 0 : WK); ++round) {
        if (wk == round) {
#pragma unroll
          for (int mi = 0; mi < MTW; ++mi) {
            const int mt = wm + WM * mi;
            if (mt < MT) {
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const int r = mt * 16 + g8 + (c >> 1) * 8;
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
      if (p.red_slots > 1) consumer_sync();
      // epilogue: bias, activation, residual (read through L2: another CTA may have written it in
      // an earlier op of this chain), bf16 RNE store
      const int nslots = p.red_slots;
      for (int q = t; q < R * N; q += kConsumers) {
        const int n = q / R, r = q - n * R;
        float v = res[(size_t)r * N + n];
        for (int w = 1; w < nslots; ++w) v += res[(size_t)w * R * N + (size_t)r * N + n];
        const long long m = row0 + r;
        if (o.bias) v += __bfloat162float(o.bias[m]);
        if (o.act == DAK_ACT_RELU) v = fmaxf(v, 0.f);
        if (o.residual) {
          const unsigned short rbits = __ldcg(reinterpret_cast<const unsigned short*>(o.residual + (long long)n * o.ldy + m));
          v += __uint_as_float((uint32_t)rbits << 16);
        }
        o.y[(long long)n * o.ldy + m] = __float2bfloat16_rn(v);
      }
      consumer_sync();  // res may be reused by the next op
      __syncwarp();
      if (lane == 0) mbar_arrive(&epi[oi]);  // this warp's y stores (and its warp-mates', via syncwarp) are done
    }
  }
}

}  // namespace chain
}  // namespace dak

// ------------------------------------------------------------------------------------ host side
namespace dak {
namespace chain {

static const int kMtwBuckets[] = {1, 2, 3, 4, 6, 8, 12};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// box = (64 elements, rows, atoms): the per-stage box (n8 rows, kc / 64 atoms) or, x-resident, the
// whole x (N rows, K / 64 atoms)
static dak_status encode_x(CUtensorMap* m, const void* x, long long N, long long K, int rows, int atoms) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    DAK_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) return fail(DAK_ECUDA, "dak_linear_chain: cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)f;
  }
  const cuuint64_t dims[3] = {64, (cuuint64_t)N, (cuuint64_t)(K / 64)};
  const cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)rows, (cuuint32_t)atoms};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DAK_ECUDA, "dak_linear_chain: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DAK_OK;
}

struct Range {
  uintptr_t b, e;
};
static bool overlap(Range a, Range b) { return a.b < b.e && b.b < a.e && a.e > a.b && b.e > b.b; }

template <int NT, int MTW, bool XRES>
static dak_status launch_t(const Params& p, int grid, int smem, cudaStream_t s, int pdl) {
  auto kern = chain_kernel<NT, MTW, XRES>;
  static int set = 0;
  if (!set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    set = 1;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  return DAK_OK;
}
template <int NT, bool XRES>
static dak_status launch_nt(const Params& p, int mtw, int grid, int smem, cudaStream_t s, int pdl) {
  switch (mtw) {
    case 1: return launch_t<NT, 1, XRES>(p, grid, smem, s, pdl);
    case 2: return launch_t<NT, 2, XRES>(p, grid, smem, s, pdl);
    case 3: return launch_t<NT, 3, XRES>(p, grid, smem, s, pdl);
    case 4: return launch_t<NT, 4, XRES>(p, grid, smem, s, pdl);
    case 6: return launch_t<NT, 6, XRES>(p, grid, smem, s, pdl);
    case 8: return launch_t<NT, 8, XRES>(p, grid, smem, s, pdl);
    case 12: return launch_t<NT, 12, XRES>(p, grid, smem, s, pdl);
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear_chain: no kernel for %d m-tiles per warp", mtw);
}

}  // namespace chain
}  // namespace dak

using namespace dak;

extern "C" {

dak_status dak_linear_chain(const dak_linear_args* ops, int32_t n_ops, void* workspace, size_t workspace_bytes,
                            dak_stream_t stream) {
  using namespace dak::chain;
  if (!ops || n_ops < 1 || n_ops > kMaxOps) return fail(DAK_EINVAL, "dak_linear_chain: 1 <= n_ops <= %d", kMaxOps);
  if (!workspace || workspace_bytes < (size_t)n_ops * sizeof(int) || !aligned16(workspace))
    return fail(DAK_EINVAL, "dak_linear_chain: workspace of >= 4 * n_ops bytes (16-byte aligned, zero-filled) needed");
  int sms = 0;
  dak_status st = dak_device_sms(&sms);
  if (st != DAK_OK) return st;
  const int grid = sms;
  const int N = ops[0].N, kc = ops[0].kc;
  if (N < 1 || N > 16) return fail(DAK_EUNSUPPORTED, "dak_linear_chain: N must be 1..16 (mma.sync path)");
  if (kc < 64 || kc > 2048 || (kc & (kc - 1))) return fail(DAK_EINVAL, "dak_linear_chain: kc must be a power of two in [64, 2048]");
  const int NT = N <= 8 ? 1 : 2, n8 = 8 * NT;
  const int KS = kc / 16, WK = KS < 8 ? KS : 8, WM = 8 / WK;
  Params p{};
  p.n_ops = n_ops;
  p.kc = kc;
  p.N = N;
  p.n8 = n8;
  p.wm = WM;
  p.wk = WK;
  p.done = (int*)workspace;
  p.evict_first = ops[0].cfg.l2_policy == 0;
  long long rmax = 1, rmax_host = 0;
  for (int i = 0; i < n_ops; ++i) {
    const dak_linear_args& a = ops[i];
    if (a.N != N || a.kc != kc) return fail(DAK_EINVAL, "dak_linear_chain: every op needs the same N and kc");
    if (a.M <= 0 || a.K <= 0 || a.K % kc || a.h < 0 || a.h > a.M) return fail(DAK_EINVAL, "dak_linear_chain: bad M / K / h of op %d", i);
    if (a.ln_w || a.x_swiglu || a.stats_out || a.cfg.cluster > 1 || (a.cfg.force_path != 0 && a.cfg.force_path != 2))
      return fail(DAK_EUNSUPPORTED, "dak_linear_chain: plain GEMV ops only (no pre-norm / SwiGLU / statistics / cluster)");
    if (!a.x || !a.y || (a.h > 0 && !a.w_host) || (a.h < a.M && !a.w_hbm) || !aligned16(a.x) || !aligned16(a.w_host) ||
        !aligned16(a.w_hbm))
      return fail(DAK_EINVAL, "dak_linear_chain: op %d pointers missing or not 16-byte aligned", i);
    if (a.act != DAK_ACT_NONE && a.act != DAK_ACT_RELU) return fail(DAK_EINVAL, "dak_linear_chain: bad act");
    Op& o = p.ops[i];
    o.w_host = (const char*)a.w_host;
    o.w_hbm = (const char*)a.w_hbm;
    o.M = a.M;
    o.K = a.K;
    o.h = a.h;
    o.ldy = a.ldy > 0 ? a.ldy : a.M;
    if (o.ldy < a.M) return fail(DAK_EINVAL, "dak_linear_chain: ldy < M");
    o.y = (__nv_bfloat16*)a.y;
    o.bias = (const __nv_bfloat16*)a.bias;
    o.residual = (const __nv_bfloat16*)a.residual;
    o.act = a.act;
    o.nchunks = (int)(a.K / kc);
    // the row partition of dak_linear (host CTAs first, contiguous ranges differing by <= 1 row)
    int nh = 0;
    if (a.h > 0) nh = (int)std::min<long long>(a.h, a.cfg.n_cta_host > 0 ? a.cfg.n_cta_host : 2);
    o.n_host = nh;
    o.n_hbm = a.h < a.M ? grid - nh : 0;
    if (o.n_hbm > a.M - a.h) o.n_hbm = (int)(a.M - a.h);
    const long long rh = nh ? (a.h + nh - 1) / nh : 0;
    const long long rg = o.n_hbm ? (a.M - a.h + o.n_hbm - 1) / o.n_hbm : 0;
    rmax = std::max(rmax, std::max(rh, rg));
    rmax_host = std::max(rmax_host, rh);
    (void)0;  // x tensor maps below, once the x mode is known
    // dependency on earlier ops of the chain: any read of op i (x, residual) or write (y) meeting an
    // earlier op's write, or a write of op i meeting an earlier op's read
    const Range xr{(uintptr_t)a.x, (uintptr_t)a.x + (uintptr_t)(N * a.K * 2)};
    const Range yr{(uintptr_t)a.y, (uintptr_t)a.y + (uintptr_t)(((N - 1) * o.ldy + a.M) * 2)};
    const Range rr{(uintptr_t)a.residual, a.residual ? (uintptr_t)a.residual + (uintptr_t)(((N - 1) * o.ldy + a.M) * 2) : 0};
    o.dep = 0;
    for (int j = 0; j < i && !o.dep; ++j) {
      const dak_linear_args& b = ops[j];
      const long long ldb = b.ldy > 0 ? b.ldy : b.M;
      const Range bx{(uintptr_t)b.x, (uintptr_t)b.x + (uintptr_t)(N * b.K * 2)};
      const Range by{(uintptr_t)b.y, (uintptr_t)b.y + (uintptr_t)(((N - 1) * ldb + b.M) * 2)};
      const Range br{(uintptr_t)b.residual, b.residual ? (uintptr_t)b.residual + (uintptr_t)(((N - 1) * ldb + b.M) * 2) : 0};
      o.dep = overlap(xr, by) || overlap(rr, by) || overlap(yr, by) || overlap(yr, bx) || overlap(yr, br);
    }
  }
  // x-resident mode when every op's whole x fits a small buffer (one TMA box: <= 256 atoms)
  long long kmax = 0;
  for (int i = 0; i < n_ops; ++i) kmax = std::max<long long>(kmax, ops[i].K);
  const bool xres = (long long)N * kmax * 2 <= 32 * 1024 && kmax / 64 <= 256;
  for (int i = 0; i < n_ops; ++i)
    if ((st = encode_x(&p.ops[i].xmap, ops[i].x, N, ops[i].K, xres ? N : n8, xres ? (int)(ops[i].K / 64) : kc / 64)) != DAK_OK)
      return st;
  // per-thread accumulator tiles: m16 tiles per warp (dak_linear's buckets)
  const long long mt_need = ((rmax + 15) / 16 + WM - 1) / WM;
  int mtw = -1;
  for (int b : kMtwBuckets)
    if (b >= mt_need) {
      mtw = b;
      break;
    }
  if (mtw < 0) return fail(DAK_EUNSUPPORTED, "dak_linear_chain: %lld rows per CTA exceed the accumulator capacity", rmax);
  const long long rows_alloc = (long long)WM * mtw * 16;
  p.red_slots = (WK > 1 && (long long)WK * rmax * N * 4 <= 48 * 1024) ? WK : 1;
  const int res_bytes = (int)(((long long)p.red_slots * rmax * N * 4 + 127) / 128 * 128);
  int pad = 0, xbytes_total;
  if (xres) {
    // stages hold exactly rmax rows; the MMA's tiles read up to rows_alloc rows, i.e. into the next
    // slot (or the pad after the ring): rows >= R are never stored
    p.w_stage_bytes = (int)(rmax * kc * 2);
    pad = (int)((rows_alloc - rmax) * kc * 2);
    p.x_stage_bytes = 0;
    p.xres_bytes = (int)(((long long)N * kmax * 2 + 2048 + 1023) / 1024 * 1024);  // + lines the garbage rows read
    xbytes_total = 2 * p.xres_bytes;
  } else {
    p.w_stage_bytes = (int)(rows_alloc * kc * 2);
    p.x_stage_bytes = n8 * kc * 2;
    p.xres_bytes = 0;
    xbytes_total = 0;
  }
  int stages = (kSmemBudget - 2048 - 1024 - res_bytes - pad - xbytes_total) / (p.w_stage_bytes + p.x_stage_bytes);
  stages = std::min(stages, kMaxStages);
  if (stages < 2) return fail(DAK_EUNSUPPORTED, "dak_linear_chain: a stage of %d B does not fit twice (use a smaller kc)",
                              p.w_stage_bytes + p.x_stage_bytes);
  p.stages = stages;
  // congestion window per op: host stages in flight per host CTA, as dak_linear sizes it
  for (int i = 0; i < n_ops; ++i) {
    const dak_launch_cfg& c = ops[i].cfg;
    Op& o = p.ops[i];
    int w = stages;
    if (o.n_host > 0) {
      const long long hs = std::max<long long>(1, (o.h + o.n_host - 1) / o.n_host * kc * 2);
      if (c.window > 0) w = std::min(c.window, stages);
      else if (c.congestion_control) {
        const long long budget = c.host_inflight_kb > 0 ? (long long)c.host_inflight_kb * 1024 : 256 * 1024;
        w = (int)std::min<long long>(stages, std::max<long long>(1, (budget + hs * o.n_host - 1) / (hs * o.n_host)));
      }
    }
    o.window = w;
  }
  p.off_x = (1024 + stages * p.w_stage_bytes + pad + 1023) / 1024 * 1024;  // 128B-swizzled boxes: 1 KB aligned
  p.res_offset = p.off_x + (xres ? xbytes_total : stages * p.x_stage_bytes);
  const int smem = p.res_offset + res_bytes + 1024;
  p.trace = trace_slot(DAK_KIND_LINEAR, ops[0].M, ops[0].K, grid);
  const int pdl = ops[0].cfg.pdl;
  if (xres)
    return NT == 1 ? launch_nt<1, true>(p, mtw, grid, smem, (cudaStream_t)stream, pdl)
                   : launch_nt<2, true>(p, mtw, grid, smem, (cudaStream_t)stream, pdl);
  return NT == 1 ? launch_nt<1, false>(p, mtw, grid, smem, (cudaStream_t)stream, pdl)
                 : launch_nt<2, false>(p, mtw, grid, smem, (cudaStream_t)stream, pdl);
}

}  // extern "C"
