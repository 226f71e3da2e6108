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
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "ptx.cuh"

#ifndef DAK_LINEAR_PART
#define DAK_LINEAR_PART 0
#endif

namespace dak {
namespace lin {

using namespace ptx;

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = 32 + kConsumers;  // warp 0 = producer
constexpr int kMaxN = 64;     // mma.sync paths
constexpr int kMaxNTc = 4096;  // tcgen05 path (one MMA covers N <= 256; two N halves up to 512; CTA groups of <= 8 up to 4096)
constexpr int kRptMax = 16;   // FMA path: rows per thread
constexpr int kMtwMax = 12;   // MMA path: m16 tiles per warp (n8 tiles <= 2; 8 for 4 n8 tiles, 4 for 8)
constexpr int kMaxStages = 16;
constexpr int kSmemBudget = 227 * 1024;

struct __align__(64) Params {
  CUtensorMap xmap;  // x [N, K] viewed as (64 elements, N rows, K/64 atoms), 128-byte swizzle
  // CTA-pair GEMM: the packed weight tiers [0 HBM, 1 host] as (64 elements, tier rows, K/64 chunks),
  // no swizzle (DAK-KC rows are stored 128B-swizzled), box (64, 128, 1); rows past the tier zero-fill
  alignas(64) CUtensorMap wmap[2];
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
  int w_stage_host, stages_host;  // host CTAs: dense slots of their (fewer) rows -> a deeper ring
  int w_stage_bytes, x_stage_bytes, n8;
  int off_x, off_ln, res_offset;  // byte offsets (from the 1024-aligned SMEM base)
  long long ldy;   // elements between consecutive rows n of y and residual
  const char* pf;  // L2 prefetch hint for the next op (nullable)
  long long pf_bytes;
  int evict_first;  // stream weights with the L2 evict_first policy
  int wm, wk;       // MMA path: consumer warps along M x along K (wm * wk == kConsumerWarps)
  int red_slots;    // MMA path: WK -> every k-warp writes its own partial slot (one barrier), 1 -> serial
  int swiglu;       // x = [gate | up] ([N, 2K]); the operand is silu(gate) * up
  int mc;           // cluster size sharing one multicast fetch of each x chunk (1: off)
  int pair;         // tcgen05, N > 512: groups of `pair` CTAs share rows, rank r computes columns [512 r, 512 r + 512)
  int wmc;          // group mode: the group is one cluster and rank 0 multicasts each W tile to all of it
  int swap;         // tcgen05 swapped operands (umma_swap_kernel): batch = MMA M, weight rows = MMA N
  int pair2;        // CTA-pair kernel (umma_pair_kernel, cta_group::2): 0 off, else batch columns per pair tile
  int p2_hp, p2_ct; // CTA-pair kernel: host-tier row pairs (256 rows each), batch-column tiles
  int kblock;       // split-K item rows (128, or 256 when swapped)
  int rgran;        // row-partition granule (1; 8 for the tcgen05 path: 8-row swizzle atoms)
  uint32_t tmem_cols;  // tcgen05 path: TMEM columns allocated (power of two >= 32)
  int ksplit;       // tcgen05 split-K: K splits (1: off); CTA = (tier row block of 128, split)
  int host_gate;    // split-K congestion control: host-item CTAs streaming at once (0: no cap)
  int k64_split;    // 64-column chunks per split
  float* part;      // split-K fp32 partials [ksplit][N][M] (workspace)
  // fused pre-norm of x (nullable ln_w): per-row statistics merged from ln_parts partials
  const __nv_bfloat16* ln_w;
  const __nv_bfloat16* ln_b;
  const float* ln_stats;
  int ln_parts;
  float ln_eps;
  int ln_rms;       // 1: RMSNorm (no mean subtraction, no bias)
  float* stats_out;  // epilogue row statistics (count, mean, M2) of this CTA's outputs (nullable)
  unsigned long long* trace;  // dak_trace_enable slot (nullable)
};

// Row range of CTA j of n in a tier of R rows, in units of g rows (sizes differ by <= one unit).
__host__ __device__ __forceinline__ void tier_rows(long long R, long long j, long long n, int g, long long* rb,
                                                   long long* re) {
  const long long U = (R + g - 1) / g;
  const long long b = (j * U / n) * g, e = ((j + 1) * U / n) * g;
  *rb = b < R ? b : R;
  *re = e < R ? e : R;
}

__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 4 + k] = t;
  }
}

// ------------------------------------------------------------------------------------ PTX glue: ptx.cuh
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
// the same, delivered to every CTA of the cluster in ctamask (same SMEM offset, each CTA's own
// mbarrier at the same offset receives the complete_tx)
__device__ __forceinline__ void tma_3d_mc(void* dst, uint64_t tmap, int c0, int c1, int c2, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;" ::
          "r"(su32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same SMEM offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(b)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Congestion control of the split-K host items (cap the SMs reading host memory). A
// split-K launch has one CTA per (128-row block, K split) item, so a large host share would put
// many host CTAs on the link at once; a counting semaphore in device memory lets at most `cap` of
// them stream, each releasing its slot once its last host stage has landed. The spin is bounded:
// a stale count can delay a launch but never hang it, and results never depend on the gate.
__device__ unsigned int g_host_gate;
__device__ __forceinline__ bool gate_acquire(int cap) {
  for (int it = 0; it < (1 << 16); ++it) {
    if (atomicAdd(&g_host_gate, 1u) < (unsigned)cap) return true;
    atomicSub(&g_host_gate, 1u);
    __nanosleep(512);
  }
  return false;
}
__device__ __forceinline__ void gate_release() {
  __threadfence();
  atomicSub(&g_host_gate, 1u);
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

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
//
// One pipeline stage = TWO copies: the CTA's (rows x KC) weight span (1-D bulk) and the x chunk
// [N8 rows x KC] (one 3-D tensor TMA, rows >= N zero-filled). Per-copy issue cost in the TMA unit
// is ~40 ns regardless of size (measured: profiles/r01/linear_copycount.txt), so the earlier
// one-bulk-copy-per-x-row scheme spent most of the TMA time on 128-512 B copies.
// x stage layout (128B swizzle): 16-byte chunk c of atom a (64 elements) of row n lives at
// ((a * N8 + n) * 128) + ((c ^ (n & 7)) << 4) -> conflict-free ldmatrix / LDS.128.
__device__ __forceinline__ uint32_t x_off(int n8, int n, int sl) {
  return (uint32_t)((((sl >> 3) * n8 + n) << 7) + (((sl & 7) ^ (n & 7)) << 4));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // identical on all lanes
  return v;
}
// LN(x) pair: ((x - mu) * rs) * w + b, rounded to bf16 (same expression as layernorm_kernel)
__device__ __forceinline__ uint32_t ln_pair(uint32_t xv, uint32_t wv, uint32_t bv, float mu, float rs) {
  float t0 = (bf_lo(xv) - mu) * rs, t1 = (bf_hi(xv) - mu) * rs;
  t0 = t0 * bf_lo(wv) + bf_lo(bv);
  t1 = t1 * bf_hi(wv) + bf_hi(bv);
  __nv_bfloat162 h = __floats2bfloat162_rn(t0, t1);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }
// SwiGLU pair: silu(gate) * up, rounded to bf16
__device__ __forceinline__ uint32_t swiglu_pair(uint32_t gv, uint32_t uv) {
  __nv_bfloat162 h = __floats2bfloat162_rn(silu_f(bf_lo(gv)) * bf_lo(uv), silu_f(bf_hi(gv)) * bf_hi(uv));
  return *reinterpret_cast<uint32_t*>(&h);
}

// XF (operand transform): 0 none, 1 fused pre-norm (LN / RMSNorm), 2 SwiGLU of [gate | up]
template <int PATH, int NN, int MTW, int XF>
__global__ void __launch_bounds__(kThreads, 1) split_linear_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128B-swizzled TMA destinations need 1024-byte alignment: align the base by hand
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* lnbar = empty + kMaxStages;
  uint64_t* xempty = lnbar + 1;  // [kMaxStages] in the cluster leader: x slot free in EVERY cluster CTA
  unsigned char* wring = smem + 1024;
  unsigned char* xring = smem + p.off_x;
  float* res = reinterpret_cast<float*>(smem + p.res_offset);

  const int cta = blockIdx.x;
  const bool host = cta < p.n_host;
  long long rb, re;  // tier-local row range
  const long long R_tier = host ? p.h : p.M - p.h;
  {
    const long long j = host ? cta : cta - p.n_host;
    const long long n = host ? p.n_host : p.n_hbm;
    tier_rows(R_tier, j, n, p.rgran, &rb, &re);
  }
  const int R = (int)(re - rb);
  const long long row0 = host ? rb : p.h + rb;  // global row of local row 0
  const char* wsrc = host ? p.w_host : p.w_hbm;
  const int slots = host ? p.window : p.stages;
  const int wstage = host ? p.w_stage_host : p.w_stage_bytes;  // W slot stride of this CTA's ring
  const int kc = p.kc;
  const int nchunks = (int)(p.K / kc);
  const int N = p.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    mbar_init(lnbar, 1);
    if (p.mc > 1)
      for (int s = 0; s < kMaxStages; ++s) mbar_init(&xempty[s], kConsumerWarps * p.mc);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t crank = p.mc > 1 ? cluster_rank() : 0u;
  if (p.mc > 1) cluster_sync();  // peers' barriers are initialised before any multicast / remote arrive
  if (threadIdx.x == 0) tstamp(p.trace, 0);
  grid_dep_launch();  // the next op may start its weight stream as our CTAs retire
  if (R <= 0) {
    if (p.stats_out && threadIdx.x < N) {
      float4* so = reinterpret_cast<float4*>(p.stats_out) + (size_t)cta * N + threadIdx.x;
      *so = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return;
  }

  const uint32_t w_bytes = (uint32_t)R * kc * 2;
  const uint32_t x_tx = (uint32_t)p.x_stage_bytes;  // the full box (zero-filled rows count)
  const long long chunk_stride = R_tier * kc * 2;  // bytes between consecutive k-chunks of a row

  if (warp == 0) {
    // ============================ producer (one lane): W span + x box per stage
    if (lane == 0) {
      const int pro = min(slots, nchunks);
      const char* src = wsrc + rb * kc * 2;
      // weights are read exactly once per step: evict_first keeps L2 for activations and for the
      // next op's prefetched prefix
      const bool ef = p.evict_first != 0;
      const uint64_t pol = policy_evict_first();
      const uint64_t xmap = reinterpret_cast<uint64_t>(&p.xmap);
      asm volatile("prefetch.tensormap [%0];" ::"l"(xmap) : "memory");
      auto load_w = [&](int slot, int i) {
        unsigned char* dst = wring + (size_t)slot * wstage;
        const char* s_ = src + (long long)i * chunk_stride;
        if (ef) bulk_g2s_hint(dst, s_, w_bytes, &full[slot], pol);
        else bulk_g2s(dst, s_, w_bytes, &full[slot]);
      };
      const uint16_t mask = (uint16_t)((1u << p.mc) - 1u);
      auto load_x = [&](int slot, int i) {
        unsigned char* dst = xring + (size_t)slot * p.x_stage_bytes;
        if (p.mc > 1) {  // the leader fetches the chunk once for the whole cluster
          if (crank != 0) return;
          tma_3d_mc(dst, xmap, 0, 0, i * (kc >> 6), &full[slot], mask);
          if (XF == 2)
            tma_3d_mc(dst + (p.x_stage_bytes >> 1), xmap, 0, 0, (int)((p.K + (long long)i * kc) >> 6), &full[slot], mask);
          return;
        }
        tma_3d(dst, xmap, 0, 0, i * (kc >> 6), &full[slot]);
        if (XF == 2) tma_3d(dst + (p.x_stage_bytes >> 1), xmap, 0, 0, (int)((p.K + (long long)i * kc) >> 6), &full[slot]);
      };
      for (int i = 0; i < pro; ++i) {  // weights do not depend on the previous kernel: start now
        mbar_expect_tx(&full[i], w_bytes + x_tx);
        load_w(i, i);
      }
      if (XF == 1) {  // LN weight / bias are parameters too: resident for the whole kernel
        const uint32_t kb = (uint32_t)p.K * 2;
        mbar_expect_tx(lnbar, p.ln_b ? 2 * kb : kb);
        bulk_g2s(smem + p.off_ln, p.ln_w, kb, lnbar);
        if (p.ln_b) bulk_g2s(smem + p.off_ln + kb, p.ln_b, kb, lnbar);
      }
      grid_dep_wait();  // x is produced by the previous kernel
      tstamp(p.trace, 1);
      for (int i = 0; i < pro; ++i) load_x(i, i);
      int s = pro == slots ? 0 : pro;
      uint32_t ph = pro == slots ? 1u : 0u;
      for (int i = pro; i < nchunks; ++i) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], w_bytes + x_tx);
        load_w(s, i);
        if (p.mc > 1 && crank == 0) mbar_wait(&xempty[s], ph ^ 1u);  // slot s free in every cluster CTA
        load_x(s, i);
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
      // this CTA's last weight copies are in flight: warm L2 with its slice of the next op's first
      // bytes so the next kernel's ramp reads L2 while this one drains (hint only)
      if (p.pf_bytes > 0) {
        const long long G = gridDim.x;
        const long long b = (p.pf_bytes * cta / G) & ~15LL;
        const long long e = (p.pf_bytes * (cta + 1) / G) & ~15LL;
        for (long long o = b; o < e; o += 32768) prefetch_l2(p.pf + o, (uint32_t)min(32768LL, e - o));
      }
    }
    __syncwarp();
    if (p.mc > 1) cluster_sync();  // peers' remote arrivals on our barriers have landed
    return;
  }

  // ================================ consumers
  const int t = threadIdx.x - 32;
  const int cw = warp - 1;
  if (p.trace && t == 0) {  // first stage landed (a second wait on a completed phase returns at once)
    mbar_wait(&full[0], 0);
    tstamp(p.trace, 2);
  }
  const uint32_t wring_u = su32(wring), xring_u = su32(xring);
  const int n8 = p.n8;
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
    uint32_t xoff[NN];
#pragma unroll
    for (int n = 0; n < NN; ++n) xoff[n] = x_off(n8, n, sl);
    float acc[RPT][NN];
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int n = 0; n < NN; ++n) acc[j][n] = 0.f;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      const unsigned char* ws = wring + (size_t)s * wstage;
      const unsigned char* xs = xring + (size_t)s * p.x_stage_bytes;
      float xf[NN][8];
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        const uint4 v = *reinterpret_cast<const uint4*>(xs + xoff[n]);
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
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        if (p.mc > 1) mbar_arrive_remote(&xempty[s], 0);  // the leader refills x for the whole cluster
      }
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
    const int WK = p.wk, WM = p.wm;
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
    // B rows: lane supplies x row n = (lane & 7) + 8 (lane >> 4), 16-byte chunk 2 ks + ((lane >> 3) & 1)
    const int bn = (lane & 7) + ((lane >> 4) << 3);
    const int bjh = (lane >> 3) & 1;
    const uint32_t b_row = (uint32_t)bn << 7;
    const uint32_t atom_bytes = (uint32_t)n8 << 7;
    // fused pre-norm: per-row mean / rstd merged from the producer's partials (count, mean, M2):
    // mean = sum c_j m_j / sum c_j, M2 = sum M2_j + c_j (m_j - mean)^2 (exact decomposition),
    // lane-strided then butterfly sums: fixed order, one warp per row n
    float mu[NT], rs[NT];
    const unsigned char* lnres = smem + p.off_ln;
    if constexpr (XF == 1) {
      grid_dep_wait();
      float* s_ln = reinterpret_cast<float*>(smem + 512);
      for (int n = cw; n < N; n += kConsumerWarps) {
        // batches of 8 independent loads per lane (one L2 round trip per 256 parts); the values
        // stay in registers for the second pass when parts <= 256 (the usual case: one per CTA)
        float c = 0.f, cm = 0.f;
        float4 v[8];
        for (int j0 = 0; j0 < p.ln_parts; j0 += 256) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = j0 + u * 32 + lane;
            v[u] = j < p.ln_parts ? *reinterpret_cast<const float4*>(p.ln_stats + ((size_t)j * N + n) * 4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            c += v[u].x;
            cm += v[u].x * v[u].y;
          }
        }
        c = warp_sum(c);
        const float mean = warp_sum(cm) / c;
        float m2 = 0.f;
        for (int j0 = 0; j0 < p.ln_parts; j0 += 256) {
          if (p.ln_parts > 256) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int j = j0 + u * 32 + lane;
              v[u] = j < p.ln_parts ? *reinterpret_cast<const float4*>(p.ln_stats + ((size_t)j * N + n) * 4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float d = v[u].y - mean;
            m2 += v[u].z + v[u].x * d * d;
          }
        }
        m2 = warp_sum(m2);
        if (lane == 0) {
          const float var = p.ln_rms ? m2 / c + mean * mean : m2 / c;  // RMS: mean of squares
          s_ln[n] = p.ln_rms ? 0.f : mean;
          s_ln[kMaxN + n] = rsqrtf(var + p.ln_eps);
        }
      }
      consumer_sync();
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n = nt * 8 + (lane >> 2);
        mu[nt] = n < N ? s_ln[n] : 0.f;
        rs[nt] = n < N ? s_ln[kMaxN + n] : 0.f;
      }
      mbar_wait(lnbar, 0);
    }
    const bool has_lnb = p.ln_b != nullptr;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      const uint32_t ws = wring_u + (uint32_t)s * wstage + a_base;
      const uint32_t xs = xring_u + (uint32_t)s * p.x_stage_bytes + b_row;
      for (int j = 0; j < nks; ++j) {
        const int ks = wk + j * WK;
        uint32_t b[NT][2];
        const int c8 = ((ks & 3) << 1) + bjh;
        const uint32_t baddr = xs + (uint32_t)(ks >> 2) * atom_bytes + (uint32_t)((c8 ^ (bn & 7)) << 4);
        if constexpr (NT == 1) {
          ldsm_x2(baddr, b[0][0], b[0][1]);
        } else {
#pragma unroll
          for (int j2 = 0; j2 < NT / 2; ++j2)  // 16 x rows per ldmatrix.x4 (+2 KB per 16 rows)
            ldsm_x4(baddr + j2 * 2048, b[2 * j2][0], b[2 * j2][1], b[2 * j2 + 1][0], b[2 * j2 + 1][1]);
        }
        if constexpr (XF == 2) {  // gate box first, up box at + x_stage_bytes / 2: silu(g) * u
          const uint32_t uaddr = baddr + (uint32_t)(p.x_stage_bytes >> 1);
          uint32_t u[NT][2];
          if constexpr (NT == 1) {
            ldsm_x2(uaddr, u[0][0], u[0][1]);
          } else {
#pragma unroll
            for (int j2 = 0; j2 < NT / 2; ++j2)
              ldsm_x4(uaddr + j2 * 2048, u[2 * j2][0], u[2 * j2][1], u[2 * j2 + 1][0], u[2 * j2 + 1][1]);
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            b[nt][0] = swiglu_pair(b[nt][0], u[nt][0]);
            b[nt][1] = swiglu_pair(b[nt][1], u[nt][1]);
          }
        }
        if constexpr (XF == 1) {  // B fragment (n = lane/4 [+8], k = 16ks + 2(lane%4) [+8]) -> LN(x)
          const int kk = i * kc + ks * 16 + 2 * (lane & 3);
          const uint32_t w0 = *reinterpret_cast<const uint32_t*>(lnres + kk * 2);
          const uint32_t w1 = *reinterpret_cast<const uint32_t*>(lnres + (kk + 8) * 2);
          const uint32_t c0 = has_lnb ? *reinterpret_cast<const uint32_t*>(lnres + (p.K + kk) * 2) : 0u;
          const uint32_t c1 = has_lnb ? *reinterpret_cast<const uint32_t*>(lnres + (p.K + kk + 8) * 2) : 0u;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            b[nt][0] = ln_pair(b[nt][0], w0, c0, mu[nt], rs[nt]);
            b[nt][1] = ln_pair(b[nt][1], w1, c1, mu[nt], rs[nt]);
          }
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
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        if (p.mc > 1) mbar_arrive_remote(&xempty[s], 0);  // the leader refills x for the whole cluster
      }
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    // deterministic cross-warp reduction over the WK warps sharing m-tiles (fixed wk order): either
    // every k-warp stores its partial into its own slot and the epilogue sums slots 0..WK-1 (one
    // barrier), or (large tiles) serial accumulation rounds in the same order
    const int g = lane >> 2, c2 = (lane & 3) * 2;
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
              const int r = mt * 16 + g + (c >> 1) * 8;
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
  // bias / residual of this thread's first two items are fetched before the reduction barrier
  float pre_b[2] = {0.f, 0.f}, pre_r[2] = {0.f, 0.f};
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int q = t + e * kConsumers;
    if (q < R * N) {
      const int n = q / R, r = q - n * R;
      const long long m = row0 + r;
      if (p.bias) pre_b[e] = __bfloat162float(p.bias[m]);
      if (p.residual) pre_r[e] = __bfloat162float(p.residual[(long long)n * p.ldy + m]);
    }
  }
  const int nslots = PATH == 2 ? p.red_slots : 1;
  if (nslots > 1) consumer_sync();
  for (int q = t; q < R * N; q += kConsumers) {
    const int n = q / R, r = q - n * R;
    float v = res[(size_t)r * RN + n];
    for (int w = 1; w < nslots; ++w) v += res[(size_t)w * R * N + (size_t)r * N + n];
    const long long m = row0 + r;
    const int e = (q - t) / kConsumers;
    if (p.bias) v += e == 0 ? pre_b[0] : (e == 1 ? pre_b[1] : __bfloat162float(p.bias[m]));
    if (p.act == DAK_ACT_RELU) v = fmaxf(v, 0.f);
    if (p.residual) v += e == 0 ? pre_r[0] : (e == 1 ? pre_r[1] : __bfloat162float(p.residual[(long long)n * p.ldy + m]));
    const __nv_bfloat16 o = __float2bfloat16_rn(v);
    p.y[(long long)n * p.ldy + m] = o;
    res[(size_t)r * RN + n] = __bfloat162float(o);  // same thread read this slot: no hazard
  }
  // row statistics of the stored outputs for a fused pre-norm in the next op (two-pass, fixed order)
  if (p.stats_out) {
    consumer_sync();
    for (int n = cw; n < N; n += kConsumerWarps) {
      float sm = 0.f;
      for (int r = lane; r < R; r += 32) sm += res[(size_t)r * RN + n];
      const float mean = warp_sum(sm) / (float)R;
      float m2 = 0.f;
      for (int r = lane; r < R; r += 32) {
        const float d = res[(size_t)r * RN + n] - mean;
        m2 += d * d;
      }
      m2 = warp_sum(m2);
      if (lane == 0)
        reinterpret_cast<float4*>(p.stats_out)[(size_t)cta * N + n] = make_float4((float)R, mean, m2, 0.f);
    }
  }
  if (p.trace) {
    consumer_sync();
    if (t == 0) tstamp(p.trace, 3);
  }
  if (p.mc > 1) cluster_sync();
}

// ------------------------------------------------------------------------------------ tcgen05 path
// PATH 3 (large N, BASELINE C3's b64 decode and beyond): the same producer and ring, but the
// dot products run on the 5th-gen tensor cores. One elected thread issues
// tcgen05.mma.cta_group::1.kind::f16 (M = 128 weight rows x N = n8 batch columns x K = 16) with
// both operands read from SMEM through descriptors, accumulating in TMEM; tcgen05.commit releases
// each ring slot; four epilogue warps move the accumulators TMEM -> registers (tcgen05.ld) for the
// bias / residual / bf16 epilogue. Operand layouts are the canonical K-major SWIZZLE_128B ones:
// KC = 64 makes a W stage rows x 128 B with 16-byte chunks XOR-swizzled by (row & 7) -- exactly
// DAK-KC when CTA row ranges start on multiples of 8 (rgran = 8) -- and the x box is the TMA's
// 128B-swizzled [n8][64]. Rows beyond R in an M = 128 tile read neighbouring SMEM; their TMEM lanes
// are never stored.
// the same arrive delivered to the mbarrier at this offset in every CTA of ctamask (cluster)
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   su32(bar)), "h"(mask)
               : "memory");
}
// 1-D bulk copy delivered to the same SMEM offset of every CTA in ctamask (each CTA's own mbarrier
// at that offset receives the complete_tx): one fetch of a weight tile for every CTA of a group
__device__ __forceinline__ void bulk_g2s_mc_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint [%0], [%1], %2, [%3], %4, %5;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "h"(mask), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// XF: operand transform as on the mma.sync path (0 none, 1 pre-norm, 2 SwiGLU), applied by three
// transform warps to each landed x box in SMEM (in place; SwiGLU writes into the gate box), made
// visible to the tensor core's async proxy, then released to the MMA issuer through xready[s].
template <int NT, int XF>  // x rows padded to n8 = 8 NT: MMA N = n8
__global__ void __launch_bounds__(kThreads, 1) umma_linear_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* done = empty + kMaxStages;
  uint64_t* xready = done + 1;  // [kMaxStages] transformed x box ready (XF != 0)
  uint64_t* lnbar = xready + kMaxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 512);
  float* s_ln = reinterpret_cast<float*>(smem + p.res_offset);  // mean[256], rstd[256] (in the slack region)
  unsigned char* wring = smem + 1024;
  unsigned char* xring = smem + p.off_x;
  constexpr int N8 = 8 * NT;
  constexpr int KCH = N8 >= 128 ? 1 : 4;  // independent k-chains (large N keeps one chain busy)

  const int cta = blockIdx.x;
  const bool host = cta < p.n_host;
  long long rb, re;
  const long long R_tier = host ? p.h : p.M - p.h;
  int kbeg = 0, kend = (int)(p.K / 64), ks = 0;  // this CTA's 64-column chunks [kbeg, kend)
  if (p.ksplit > 1) {  // split-K: (128-row block, K split) per CTA; splits fixed by (M, K)
    const int j = host ? cta : cta - p.n_host;
    ks = j % p.ksplit;
    rb = (long long)(j / p.ksplit) * 128;
    re = rb + 128 < R_tier ? rb + 128 : R_tier;
    kbeg = ks * p.k64_split;
    kend = kbeg + p.k64_split < kend ? kbeg + p.k64_split : kend;
  } else if (N8 > 256 && p.pair > 1) {  // CTA groups: every rank takes the group's rows
    tier_rows(R_tier, (host ? cta : cta - p.n_host) / p.pair, (host ? p.n_host : p.n_hbm) / p.pair, p.rgran, &rb, &re);
  } else {
    tier_rows(R_tier, host ? cta : cta - p.n_host, host ? p.n_host : p.n_hbm, p.rgran, &rb, &re);
  }
  const int G = (N8 > 256 && p.pair > 1) ? p.pair : 1;  // CTAs per group
  const int prank = cta % G;  // group rank = cluster rank (groups start at multiples of G)
  const bool wmc = G > 1 && p.wmc;
  const int R = (int)(re - rb);
  const long long row0 = host ? rb : p.h + rb;
  const char* wsrc = host ? p.w_host : p.w_hbm;
  const int slots = host ? p.window : p.stages;
  const int wstage = host ? p.w_stage_host : p.w_stage_bytes;
  const int nchunks = kend - kbeg;
  const int N = p.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtiles = (R + 127) >> 7;
  const uint32_t tcols = p.tmem_cols;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], wmc && prank == 0 ? G : 1);  // W multicast: rank 0 refills after ALL consumed
    }
    mbar_init(done, 1);
    for (int s = 0; s < kMaxStages; ++s) mbar_init(&xready[s], 3);  // three transform warps
    mbar_init(lnbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1 && R > 0) {  // TMEM accumulator: mtiles x N8 columns (power of two >= 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wmc) cluster_sync_all();  // the peer's barrier inits are visible before any multicast / remote arrive
  if (threadIdx.x == 0) tstamp(p.trace, 0);
  grid_dep_launch();
  if (R <= 0) {
    if (p.stats_out && threadIdx.x < N)
      reinterpret_cast<float4*>(p.stats_out)[(size_t)cta * N + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const uint32_t tmem = *tslot;
  const uint32_t w_bytes = (uint32_t)R * 128;
  const uint32_t x_tx = (uint32_t)p.x_stage_bytes;
  const long long chunk_stride = R_tier * 128;

  if (warp == 0) {
    if (lane == 0) {  // producer: W span + x box per 64-column stage
      const int pro = min(slots, nchunks);
      const char* src = wsrc + rb * 128 + (long long)kbeg * chunk_stride;
      const uint64_t pol = policy_evict_first();
      const uint64_t xmap = reinterpret_cast<uint64_t>(&p.xmap);
      asm volatile("prefetch.tensormap [%0];" ::"l"(xmap) : "memory");
      // W tile of a stage: own copy, or (group + multicast) rank 0 fetches it once for all G CTAs;
      // every CTA's full barrier expects the W bytes either way
      auto load_w = [&](int slot, int i) {
        if (!wmc) bulk_g2s_hint(wring + (size_t)slot * wstage, src + (long long)i * chunk_stride, w_bytes, &full[slot], pol);
        else if (prank == 0)
          bulk_g2s_mc_hint(wring + (size_t)slot * wstage, src + (long long)i * chunk_stride, w_bytes, &full[slot],
                           (uint16_t)((1u << G) - 1u), pol);
      };
      // gated host items wait for the previous kernel first: a slot held across griddepcontrol.wait
      // would block that kernel's own host items (programmatic dependent launch overlaps the two)
      if (host && p.host_gate > 0) grid_dep_wait();
      const bool gated = host && p.host_gate > 0 && gate_acquire(p.host_gate);
      for (int i = 0; i < pro; ++i) {
        mbar_expect_tx(&full[i], w_bytes + x_tx);
        load_w(i, i);
      }
      grid_dep_wait();
      tstamp(p.trace, 1);
      if (XF == 1) {  // LN weight (+ bias) resident for the whole kernel
        const uint32_t kb = (uint32_t)p.K * 2;
        mbar_expect_tx(lnbar, p.ln_b ? 2 * kb : kb);
        bulk_g2s(smem + p.off_ln, p.ln_w, kb, lnbar);
        if (p.ln_b) bulk_g2s(smem + p.off_ln + kb, p.ln_b, kb, lnbar);
      }
      auto load_x = [&](int slot, int i) {
        unsigned char* dst = xring + (size_t)slot * p.x_stage_bytes;
        tma_3d(dst, xmap, 0, 512 * prank, kbeg + i, &full[slot]);
        if constexpr (N8 > 256) tma_3d(dst + 256 * 128, xmap, 0, 512 * prank + 256, kbeg + i, &full[slot]);  // 2nd box
        if (XF == 2) tma_3d(dst + (p.x_stage_bytes >> 1), xmap, 0, 0, (int)((p.K >> 6) + kbeg + i), &full[slot]);
      };
      for (int i = 0; i < pro; ++i) load_x(i, i);
      int s = pro == slots ? 0 : pro;
      uint32_t ph = pro == slots ? 1u : 0u;
      int ls = pro - 1;
      uint32_t lph = 0;
      for (int i = pro; i < nchunks; ++i) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], w_bytes + x_tx);
        load_w(s, i);
        load_x(s, i);
        ls = s;
        lph = ph;
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
      if (gated) {  // the last host stage has landed: free the link slot
        mbar_wait(&full[ls], lph);
        gate_release();
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the ring (converged), one elected lane issues
    {
      // kind::f16 instruction descriptor: D f32, A / B bf16, both K-major, N = N8, M = 128
      constexpr int NI = N8 > 256 ? 256 : N8;  // N per instruction (N8 = 512: two halves of 256 columns)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NI >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t wr = su32(wring), xr = su32(xring);
      uint32_t leader;
      asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nchunks; ++i) {
        mbar_wait(XF ? &xready[s] : &full[s], ph);
        tc_fence_after();
        if (leader) {
          const uint32_t ws = wr + (uint32_t)s * wstage, xs = xr + (uint32_t)s * p.x_stage_bytes;
          // 4 x K=16 per 128-byte row, each k-step into its OWN accumulator: consecutive MMAs into
          // one accumulator form a dependent chain (~140 cycles each, measured) that small-N tiles
          // cannot hide; four independent chains are summed in fixed order by the epilogue
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = umma_desc_sw128(xs + k * 32);
            for (int mt = 0; mt < mtiles; ++mt)
              umma_bf16(tmem + (uint32_t)(((k % KCH) * mtiles + mt) * N8), umma_desc_sw128(ws + mt * 128 * 128 + k * 32),
                        bd, idesc, (KCH == 4 ? i : (i | k)) != 0);
            if constexpr (N8 > 256)  // columns 256..511: x rows 256.. (second box, 32 KB on), TMEM +256
              umma_bf16(tmem + 256u, umma_desc_sw128(ws + k * 32), umma_desc_sw128(xs + 256 * 128 + k * 32), idesc,
                        (i | k) != 0);
          }
          if (wmc && prank > 0) umma_commit_mc(&empty[s], (uint16_t)(1u | (1u << prank)));  // own + rank 0's slot s
          else umma_commit(&empty[s]);  // the slot is free once these MMAs have read it
        }
        __syncwarp();
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
      if (leader) umma_commit(done);
      __syncwarp();
    }
  } else if (XF != 0 && (warp == 2 || warp == 3 || warp == 8)) {
    const int tw = warp == 8 ? 2 : warp - 2;  // transform warp 0..2
    const int tt = tw * 32 + lane;             // 0..95
    if constexpr (XF == 1) {  // per-row mean / rstd from the producer's partials (as on path 2)
      grid_dep_wait();
      for (int n = tw; n < N; n += 3) {
        float c = 0.f, cm = 0.f;
        for (int j = lane; j < p.ln_parts; j += 32) {
          const float4 v = *reinterpret_cast<const float4*>(p.ln_stats + ((size_t)j * N + n) * 4);
          c += v.x;
          cm += v.x * v.y;
        }
        c = warp_sum(c);
        const float mean = warp_sum(cm) / c;
        float m2 = 0.f;
        for (int j = lane; j < p.ln_parts; j += 32) {
          const float4 v = *reinterpret_cast<const float4*>(p.ln_stats + ((size_t)j * N + n) * 4);
          const float d = v.y - mean;
          m2 += v.z + v.x * d * d;
        }
        m2 = warp_sum(m2);
        if (lane == 0) {
          const float var = p.ln_rms ? m2 / c + mean * mean : m2 / c;
          s_ln[n] = p.ln_rms ? 0.f : mean;
          s_ln[256 + n] = rsqrtf(var + p.ln_eps);
        }
      }
      asm volatile("bar.sync 3, 96;" ::: "memory");
      mbar_wait(lnbar, 0);
    }
    const unsigned char* lnres = smem + p.off_ln;
    const bool has_lnb = p.ln_b != nullptr;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      unsigned char* xs = xring + (size_t)s * p.x_stage_bytes;
      // 16-byte chunk c of row n sits at n * 128 + ((c ^ (n & 7)) << 4): elements k = 64 i + 8 c ..
      for (int q = tt; q < N8 * 8; q += 96) {
        const int n = q >> 3, c = q & 7;
        uint4* g = reinterpret_cast<uint4*>(xs + n * 128 + ((c ^ (n & 7)) << 4));
        uint4 v = *g;
        if constexpr (XF == 2) {
          const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(g) + (p.x_stage_bytes >> 1));
          v.x = swiglu_pair(v.x, u.x); v.y = swiglu_pair(v.y, u.y);
          v.z = swiglu_pair(v.z, u.z); v.w = swiglu_pair(v.w, u.w);
        } else {
          const float mu = n < N ? s_ln[n] : 0.f, rs = n < N ? s_ln[256 + n] : 0.f;
          const int k0 = (kbeg + i) * 64 + c * 8;
          const uint4 wv = *reinterpret_cast<const uint4*>(lnres + k0 * 2);
          const uint4 bv = has_lnb ? *reinterpret_cast<const uint4*>(lnres + (p.K + k0) * 2) : make_uint4(0, 0, 0, 0);
          v.x = ln_pair(v.x, wv.x, bv.x, mu, rs); v.y = ln_pair(v.y, wv.y, bv.y, mu, rs);
          v.z = ln_pair(v.z, wv.z, bv.z, mu, rs); v.w = ln_pair(v.w, wv.w, bv.w, mu, rs);
        }
        *g = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&xready[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  } else if (warp >= 4 && warp < 8) {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = rows of the M tile. One thread polls
    // `done` with back-off, the others sleep on a named barrier: 128 threads spinning on an
    // mbarrier for the whole kernel slowed the producer / MMA barrier traffic 3x (measured).
    if (threadIdx.x == 128) {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(su32(done)), "r"(0u)
            : "memory");
        if (!ok) __nanosleep(256);
      }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    tc_fence_after();
    grid_dep_wait();  // residual / y may belong to the previous kernel
    const int q = warp & 3;
    // row statistics (stats_out): per column, this warp's rows summed (sum, sum of squares, fixed
    // butterfly order), the four warps combined in order; M2 = sumsq - R mean^2 (R <= 256 rows)
    float* st_part = s_ln + 512;  // [4 warps][N8][2] in the slack region
#pragma unroll 1
    for (int c0 = 0; c0 < N8; c0 += 8) {
      float ssum[8], ssq[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) ssum[e] = ssq[e] = 0.f;
      for (int mt = 0; mt < mtiles; ++mt) {
        const int r = mt * 128 + 32 * q + lane;
        const long long m = row0 + r;
        const float bias = (r < R && p.bias) ? __bfloat162float(p.bias[m]) : 0.f;
        float acc[8];
#pragma unroll
        for (int k = 0; k < KCH; ++k) {  // fixed-order sum of the k-chains
          uint32_t v[8];
          tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)((k * mtiles + mt) * N8 + c0), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = k == 0 ? __uint_as_float(v[e]) : acc[e] + __uint_as_float(v[e]);
        }
        if (p.ksplit > 1) {  // raw fp32 partial; bias / act / residual in splitk_reduce_kernel
          if (r < R) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int n = c0 + e;
              if (n < N) p.part[((size_t)ks * N + n) * p.M + m] = acc[e];
            }
          }
          continue;
        }
        if (r < R) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int n = 512 * prank + c0 + e;  // group rank r owns columns 512 r ..
            if (n < N) {
              float o = acc[e] + bias;
              if (p.act == DAK_ACT_RELU) o = fmaxf(o, 0.f);
              if (p.residual) o += __bfloat162float(p.residual[(long long)n * p.ldy + m]);
              const __nv_bfloat16 ob = __float2bfloat16_rn(o);
              p.y[(long long)n * p.ldy + m] = ob;
              const float f = __bfloat162float(ob);
              ssum[e] += f;
              ssq[e] += f * f;
            }
          }
        }
      }
      if (p.stats_out) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float a = warp_sum(ssum[e]), b2 = warp_sum(ssq[e]);
          if (lane == 0) {
            st_part[(q * N8 + c0 + e) * 2 + 0] = a;
            st_part[(q * N8 + c0 + e) * 2 + 1] = b2;
          }
        }
      }
    }
    if (p.stats_out) {
      asm volatile("bar.sync 2, 128;" ::: "memory");
      for (int n = threadIdx.x - 128; n < N; n += 128) {
        float a = 0.f, b2 = 0.f;
        for (int w = 0; w < 4; ++w) {
          a += st_part[(w * N8 + n) * 2 + 0];
          b2 += st_part[(w * N8 + n) * 2 + 1];
        }
        const float mean = a / (float)R;
        const float m2 = fmaxf(b2 - (float)R * mean * mean, 0.f);
        reinterpret_cast<float4*>(p.stats_out)[(size_t)cta * N + n] = make_float4((float)R, mean, m2, 0.f);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (wmc) cluster_sync_all();  // neither CTA exits while its peer may still arrive on its barriers
  if (threadIdx.x == 32 && p.trace) tstamp(p.trace, 3);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
}


#if DAK_LINEAR_PART == 5
// Swapped-operand tcgen05 split GEMM for decode batches (N <= 128), split K: the batch is the MMA's
// M side (x box of 128 rows, TMA zero-fills rows >= N) and the weight rows are its N side (up to 256
// per instruction). A kind::f16 MMA costs ~100 cycles for any N <= 128 and 128 at N = 256
// (profiles/r01/umma_micro.txt), so 256 weight rows per instruction move twice the weight bytes per
// MMA of the M = 128 weight-tile form. CTA = (block of kblock <= 256 rows of one tier, K split);
// D[batch row][weight row] in TMEM, epilogue warp q reads lanes 32q.. (batch rows) and writes the
// fp32 partial part[s][n][m] (8 consecutive m per load). Summation order of a row: fixed by the
// split (S from M, K only) -- independent of the tier split (bitwise r-invariant).
__global__ void __launch_bounds__(kThreads, 1) umma_swap_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* done = empty + kMaxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 512);
  unsigned char* wring = smem + 1024;
  unsigned char* xring = smem + p.off_x;
  const int cta = blockIdx.x;
  const bool host = cta < p.n_host;
  const long long R_tier = host ? p.h : p.M - p.h;
  const int j = host ? cta : cta - p.n_host;
  const int ks = j % p.ksplit;
  const long long rb = (long long)(j / p.ksplit) * p.kblock;
  const long long re = rb + p.kblock < R_tier ? rb + p.kblock : R_tier;
  const int kbeg = ks * p.k64_split;
  const int kend = min(kbeg + p.k64_split, (int)(p.K / 64));
  const int R = (int)(re - rb);
  const long long row0 = host ? rb : p.h + rb;
  const char* wsrc = host ? p.w_host : p.w_hbm;
  const int slots = host ? p.window : p.stages;
  const int nchunks = kend - kbeg;
  const int N = p.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tcols = p.tmem_cols;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1 && R > 0 && nchunks > 0) {  // (the same condition as the early return below: no leak)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) tstamp(p.trace, 0);
  grid_dep_launch();
  if (R <= 0 || nchunks <= 0) return;
  const uint32_t tmem = *tslot;
  const uint32_t w_bytes = (uint32_t)R * 128;
  const uint32_t x_tx = (uint32_t)p.x_stage_bytes;
  const long long chunk_stride = R_tier * 128;
  const int wstage = p.w_stage_bytes;
  if (warp == 0) {
    if (lane == 0) {  // producer: W span + x box per 64-column stage
      const int pro = min(slots, nchunks);
      const char* src = wsrc + rb * 128 + (long long)kbeg * chunk_stride;
      const uint64_t pol = policy_evict_first();
      const uint64_t xmap = reinterpret_cast<uint64_t>(&p.xmap);
      asm volatile("prefetch.tensormap [%0];" ::"l"(xmap) : "memory");
      if (host && p.host_gate > 0) grid_dep_wait();  // never hold a slot across the dependency wait
      const bool gated = host && p.host_gate > 0 && gate_acquire(p.host_gate);
      for (int i = 0; i < pro; ++i) {
        mbar_expect_tx(&full[i], w_bytes + x_tx);
        bulk_g2s_hint(wring + (size_t)i * wstage, src + (long long)i * chunk_stride, w_bytes, &full[i], pol);
      }
      grid_dep_wait();
      tstamp(p.trace, 1);
      for (int i = 0; i < pro; ++i) tma_3d(xring + (size_t)i * p.x_stage_bytes, xmap, 0, 0, kbeg + i, &full[i]);
      int s = pro == slots ? 0 : pro;
      uint32_t ph = pro == slots ? 1u : 0u;
      int ls = pro - 1;
      uint32_t lph = 0;
      for (int i = pro; i < nchunks; ++i) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], w_bytes + x_tx);
        bulk_g2s_hint(wring + (size_t)s * wstage, src + (long long)i * chunk_stride, w_bytes, &full[s], pol);
        tma_3d(xring + (size_t)s * p.x_stage_bytes, xmap, 0, 0, kbeg + i, &full[s]);
        ls = s;
        lph = ph;
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
      if (gated) {  // the last host stage has landed: free the link slot
        mbar_wait(&full[ls], lph);
        gate_release();
      }
    }
  } else if (warp == 1) {  // MMA issuer: D[128 batch rows][RN weight rows] += x . W^T
    const int RN = (R + 15) & ~15;  // M = 128 needs N % 16 == 0 (rows past R: ignored columns)
    const uint32_t MM = p.swap == 2 ? 64u : 128u;  // batch <= 64: M = 64 (x box of 64 rows)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(RN >> 3) << 17) | ((MM >> 4) << 24);
    const uint32_t wr = su32(wring), xr = su32(xring);
    uint32_t leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (leader) {
        const uint32_t ws = wr + (uint32_t)s * wstage, xs = xr + (uint32_t)s * p.x_stage_bytes;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem, umma_desc_sw128(xs + k * 32), umma_desc_sw128(ws + k * 32), idesc, (i | k) != 0);
        umma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    if (leader) umma_commit(done);
    __syncwarp();
  }
  // ---- epilogue (every warp): TMEM -> SMEM tile -> coalesced fp32 partial part[ks][n][row0..row0+R)
  if (threadIdx.x == 0) {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(su32(done)), "r"(0u)
          : "memory");
      if (!ok) __nanosleep(128);
    }
  }
  __syncthreads();  // every MMA has completed, so every ring stage has landed and been read: the ring is free
  tc_fence_after();
  grid_dep_wait();  // the partial buffer may still be read by the previous kernel
  const int RN = (R + 15) & ~15;
  const int pitch = RN + 4;  // floats; +16 B per row: 2-way bank conflicts at most on the tile stores
  float* tile = reinterpret_cast<float*>(wring);
  {
    // warp w reads TMEM lane quadrant q = w & 3 (tcgen05.ld lane restriction) and half of the
    // 16-column groups. M = 128: TMEM lane 32q + l holds batch row 32q + l. M = 64 (measured,
    // tools/umma_m64_layout.cu): batch row r sits in lane 32 (r / 16) + r % 16.
    const int q = warp & 3, half = (warp >> 2) & 1;
    const int n = p.swap == 2 ? (lane < 16 ? 16 * q + lane : -1) : 32 * q + lane;
    const int G = RN / 16, g0 = half ? G / 2 : 0, g1 = warp >= 8 ? 0 : (half ? G : G / 2);  // warp 8: idle
#pragma unroll 1
    for (int g = g0; g < g1; ++g) {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(16 * g), v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (n >= 0 && n < N) {
        float4* d4 = reinterpret_cast<float4*>(tile + (size_t)n * pitch + 16 * g);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          d4[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]), __uint_as_float(v[4 * e + 2]),
                              __uint_as_float(v[4 * e + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  const int R4 = R >> 2;  // R % 4 == 0 (M % 4 == 0, h % 8 == 0, kblock % 8 == 0)
  {
    float* dst = p.part + (size_t)ks * N * p.M + row0;
    for (int i = threadIdx.x; i < N * R4; i += kThreads) {
      const int nn = i / R4, m4 = i - nn * R4;
      __stcg(reinterpret_cast<float4*>(dst + (size_t)nn * p.M) + m4,
             *reinterpret_cast<const float4*>(tile + (size_t)nn * pitch + 4 * m4));
    }
  }
  __syncthreads();
  if (threadIdx.x == 32 && p.trace) tstamp(p.trace, 3);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
}
#endif

#if DAK_LINEAR_PART == 0
// y[n, m] = act(sum_s part[s][n][m] + bias[m]) + residual[n, m]: the fixed-order split-K combine.
// Grid (x: column groups, y: row n); vec = 4 columns per thread (float4 partial loads, 8-byte
// bf16 stores; M % 4 == 0 and 8-byte aligned y / residual rows), else one.
__device__ __forceinline__ void tstamp2d(unsigned long long* tr, int k) {  // 2-D grid: CTA = y * gridDim.x + x
  const unsigned c = blockIdx.y * gridDim.x + blockIdx.x;
  if (tr && threadIdx.x == 0 && c < (unsigned)kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[c * 4 + k] = t;
  }
}
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int S, int N, long long M,
                                     const __nv_bfloat16* __restrict__ bias, int act,
                                     const __nv_bfloat16* residual, __nv_bfloat16* y, long long ldy, int vec,
                                     unsigned long long* tr) {
  tstamp2d(tr, 0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tstamp2d(tr, 1);
  const long long total = (long long)N * M;
  const int n = blockIdx.y;
  const float* pr = part + (long long)n * M;
  __nv_bfloat16* yr = y + (long long)n * ldy;
  const __nv_bfloat16* rr = residual ? residual + (long long)n * ldy : nullptr;
  if (vec) {
    for (long long m4 = (long long)blockIdx.x * blockDim.x + threadIdx.x; m4 < M / 4; m4 += (long long)gridDim.x * blockDim.x) {
      float4 v = reinterpret_cast<const float4*>(pr)[m4];
      for (int s = 1; s < S; ++s) {
        const float4 t = reinterpret_cast<const float4*>(pr + (long long)s * total)[m4];
        v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w;
      }
      float f[4] = {v.x, v.y, v.z, v.w};
      if (bias) {
        const uint2 bb = reinterpret_cast<const uint2*>(bias)[m4];
        const float2 b0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bb.x));
        const float2 b1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bb.y));
        f[0] += b0.x; f[1] += b0.y; f[2] += b1.x; f[3] += b1.y;
      }
      if (act == DAK_ACT_RELU)
        for (int i = 0; i < 4; ++i) f[i] = fmaxf(f[i], 0.f);
      if (rr) {
        const uint2 rb = reinterpret_cast<const uint2*>(rr)[m4];
        const float2 r0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rb.x));
        const float2 r1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rb.y));
        f[0] += r0.x; f[1] += r0.y; f[2] += r1.x; f[3] += r1.y;
      }
      __nv_bfloat162 o0 = __floats2bfloat162_rn(f[0], f[1]), o1 = __floats2bfloat162_rn(f[2], f[3]);
      uint2 ob;
      ob.x = *reinterpret_cast<uint32_t*>(&o0);
      ob.y = *reinterpret_cast<uint32_t*>(&o1);
      reinterpret_cast<uint2*>(yr)[m4] = ob;
    }
    tstamp2d(tr, 3);
    return;
  }
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (long long)gridDim.x * blockDim.x) {
    float v = pr[m];
    for (int s = 1; s < S; ++s) v += pr[(long long)s * total + m];
    if (bias) v += __bfloat162float(bias[m]);
    if (act == DAK_ACT_RELU) v = fmaxf(v, 0.f);
    if (rr) v += __bfloat162float(rr[m]);
    yr[m] = __float2bfloat16_rn(v);
  }
  tstamp2d(tr, 3);
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

#endif

// ------------------------------------------------------------------------------------ host side
struct Plan {
  Params p;
  int path, nn, bucket, grid, smem;
  long long rmax_host, rmax_hbm;
};

// Clusters of `mc` one-CTA-per-SM blocks the device co-schedules at once (GPCs with an odd number
// of usable SMs leave SMs idle): the multicast grid is sized to this, never to a second wave.
template <int PATH, int NN, int MTW, int XF>
__global__ void split_linear_kernel(const __grid_constant__ Params p);
static dak_status max_active_clusters(int mc, int* out) {
  static int cache[5] = {0, 0, 0, 0, 0};
  if (mc < 1 || mc > 4) return fail(DAK_EINVAL, "dak_linear: bad cluster size");
  if (cache[mc] <= 0) {
    auto kern = split_linear_kernel<1, 1, 1, 0>;
    DAK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(mc * 64);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 200 * 1024;  // any size forcing one CTA per SM
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    DAK_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg));
    cache[mc] = n;
  }
  *out = cache[mc];
  return DAK_OK;
}

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

// compiled m16-tile buckets per warp for each n8-tile count (accumulators: MTW x NT x 4 registers)
static int mtw_max_for(int nt) { return nt <= 2 ? 12 : (nt == 4 ? 8 : 4); }

// Rows a CTA may own for a given KC (accumulator capacity of each path).
static long long path_row_cap(int path, int kc, int nt) {
  if (path == 1) {
    const int S = kc / 8;
    return (long long)(kConsumers / S) * kRptMax;
  }
  const int KS = kc / 16;
  const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
  return 16LL * (kConsumerWarps / WK) * mtw_max_for(nt);
}

static dak_status make_plan(const dak_linear_args* a, Plan* out) {
  if (!a) return fail(DAK_EINVAL, "dak_linear: args NULL");
  const long long M = a->M, K = a->K, h = a->h;
  const int N = a->N, kc = a->kc;
  if (M <= 0 || K <= 0 || N <= 0) return fail(DAK_EINVAL, "dak_linear: M, K, N must be positive");
  if (h < 0 || h > M) return fail(DAK_EINVAL, "dak_linear: h must be in [0, M]");
  if (N > kMaxNTc) return fail(DAK_EUNSUPPORTED, "dak_linear: N=%d > %d", N, kMaxNTc);
  // n8 tiles (compiled: 1, 2, 4, 8 on every path; 16, 32 on the tcgen05 path)
  const int nt = N <= 8 ? 1 : (N <= 16 ? 2 : (N <= 32 ? 4 : (N <= 64 ? 8 : (N <= 128 ? 16 : (N <= 256 ? 32 : 64)))));
  // N > 512: groups of G = ceil(N / 512) CTAs over the same rows (rank r: columns [512 r, 512 r + 512));
  // CTA counts below are groups
  const int G = N > 512 ? (N + 511) / 512 : 1;
  const bool pair = G > 1;
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
  // default: tensor cores for every N -- mma.sync (path 2) up to N = 16; tcgen05 (path 3) beyond,
  // where mma.sync becomes issue-bound, when its operand constraints hold
  int path = c.force_path ? c.force_path : 2;
  // 9..16 columns: tcgen05 too when every CTA owns >= 128 rows (one M = 128 tile, no split-K) --
  // mma.sync's two n8 tiles per k-step become issue-bound there (OPT-30B qkv / fc1 / head at b16)
  bool tc_n16 = false;
  if (!c.force_path && N > 8 && N <= 16 && kc == 64) {
    int sm = 0;
    dak_status st = device_sms(&sm);
    if (st != DAK_OK) return st;
    tc_n16 = M >= 128LL * sm;
  }
  if (!c.force_path && (N > 16 || tc_n16) && kc == 64 && (c.cluster <= 1 || N > 512) && h % 8 == 0)  // cluster at N > 512: W multicast groups
    path = 3;
  if (path == 1 && N > 4) return fail(DAK_EUNSUPPORTED, "dak_linear: CUDA-core path supports N <= 4");
  const bool force_swap = path == 4;  // force_path 4: tcgen05 with swapped operands (split-K decode form)
  if (force_swap) path = 3;
  const bool force_pair = path == 5;  // force_path 5: the CTA-pair (cta_group::2) GEMM
  if (force_pair) path = 3;
  if (path != 1 && path != 2 && path != 3) return fail(DAK_EINVAL, "dak_linear: bad force_path");
  if (path != 3 && N > kMaxN) return fail(DAK_EUNSUPPORTED, "dak_linear: N=%d > %d needs the tcgen05 path (kc = 64)", N, kMaxN);
  if (path == 3) {  // tcgen05: canonical SWIZZLE_128B K-major operands need KC = 64; plain GEMV only
    if (kc != 64) return fail(DAK_EUNSUPPORTED, "dak_linear: the tcgen05 path needs kc = 64");
  }
  const int nt_eff = path == 3 ? std::max(2, nt) : nt;  // tcgen05 M = 128 needs N >= 16
  const int rg = path == 3 ? 8 : 1;                     // 8-row swizzle atoms per CTA range
  // rows per CTA are bounded by the accumulator capacity of the path and by SMEM: at least three
  // ring stages of (rows x KC) weights plus the x rows must fit (deep enough to cover HBM latency)
  if (a->x_swiglu && (path == 1 || a->ln_w)) return fail(DAK_EINVAL, "dak_linear: x_swiglu needs a tensor-core path and no pre-norm");
  const int n8 = path == 1 ? 8 : nt_eff * 8;
  const long long x_stage = (long long)n8 * kc * 2 * (a->x_swiglu ? 2 : 1);
  // N > 256 (tcgen05, 512 TMEM columns): one M tile per CTA, a 64 KB x box per stage, two stages
  const bool wide = path == 3 && n8 > 256;
  if (wide && (a->ln_w || a->x_swiglu || a->stats_out))
    return fail(DAK_EUNSUPPORTED, "dak_linear: N > 256 supports the plain GEMM only (no pre-norm / SwiGLU / statistics)");
  const long long smem_rows = wide ? ((kSmemBudget - 2048 - 16384) / 2 - x_stage) / (kc * 2) / 16 * 16
                                   : ((kSmemBudget - 2048 - 8192) / 3 - x_stage) / (kc * 2) / 16 * 16;
  if (path == 1 && kc > 8 * kConsumers) return fail(DAK_EUNSUPPORTED, "dak_linear: CUDA-core path needs kc <= %d", 8 * kConsumers);
  const long long cap = std::min(path == 3 ? (wide ? 128LL : 256LL) : path_row_cap(path, kc, nt), smem_rows);
  if (cap < 16) return fail(DAK_EUNSUPPORTED, "dak_linear: kc=%d leaves no room for a 16-row stage", kc);

  int n_host = 0;
  if (h > 0) {
    n_host = c.n_cta_host > 0 ? c.n_cta_host : 2;  // 2 CTAs saturate the link (calibration)
    n_host = (int)std::max<long long>(n_host, ceil_div(h, cap));
    n_host = (int)std::min<long long>(n_host, h);
  }
  int n_hbm = 0;
  if (h < M) {
    n_hbm = c.n_cta_hbm > 0 ? c.n_cta_hbm : std::max(1, sms / G - n_host);
    n_hbm = (int)std::max<long long>(n_hbm, ceil_div(M - h, cap));
    n_hbm = (int)std::min<long long>(n_hbm, M - h);
  }
  // x multicast: clusters of mc CTAs never mix tiers and every CTA owns >= 1 row (else off)
  int mc = c.cluster > 1 ? c.cluster : 1;
  if (mc != 1 && mc != 2 && mc != 4) return fail(DAK_EINVAL, "dak_linear: cluster must be 0, 1, 2 or 4");
  if (mc > 1 && path != 2) mc = 1;
  if (rg > 1) {  // every CTA owns whole 8-row units
    n_host = (int)std::min<long long>(n_host, ceil_div(h, rg));
    n_hbm = (int)std::min<long long>(n_hbm, ceil_div(M - h, rg));
    if (h > 0 && h % rg && !force_pair) return fail(DAK_EINVAL, "dak_linear: the tcgen05 path needs h %% 8 == 0");
  }
  if (mc > 1) {
    const int nh2 = n_host ? (int)ceil_div(n_host, mc) * mc : 0;
    int ng2 = n_hbm ? std::max(mc, n_hbm / mc * mc) : 0;
    if (n_hbm && c.n_cta_hbm <= 0) {  // auto grid: only as many clusters as run concurrently
      int clusters = 0;
      dak_status st = max_active_clusters(mc, &clusters);
      if (st != DAK_OK) return st;
      ng2 = std::max(mc, std::min(ng2, (clusters - nh2 / mc) * mc));
    }
    if (nh2 <= h && ng2 <= M - h && (!n_host || ceil_div(h, nh2) <= cap) && (!n_hbm || ceil_div(M - h, ng2) <= cap)) {
      n_host = nh2;
      n_hbm = ng2;
    } else {
      mc = 1;
    }
  }
  // tcgen05 split-K: an M = 128 tile costs the same time however few of its rows are real, so when
  // the auto partition leaves < 128 rows per CTA, CTAs take (128-row block, K split) items instead;
  // splits are fixed by (M, K, SM count), never by the tier split h, keeping every row's summation order
  // independent of the tier split (bitwise r-invariance). Needs caller workspace for the partials.
  int ksplit = 1, k64_split = (int)(K / 64), swap = 0, kblock = 128;
  if (path == 3 && !pair && !a->stats_out && !a->ln_w && !a->x_swiglu && c.n_cta_hbm <= 0 && a->workspace) {
    // S from (M, K, SM count) only: as many splits as keep all items in ONE wave (even if h adds a
    // tile). Measured at the Llama TP8 b64 shapes (profiles/r01/splitk_sweep.txt): a second wave or
    // shorter splits cost more than the idle SMs of a partial wave.
    const long long C = K / 64, nsm = std::max(1, sms);
    long long S = std::min<long long>(std::min<long long>(16, C), nsm / (ceil_div(M, 128) + 1));
    long long bks = C;
    if (S > 1) {
      bks = ceil_div(C, S);
      S = ceil_div(C, bks);
    }
    if (S > 1 && ceil_div(M, nsm) < 128) {  // from M and the SM count only (never h: r-invariance)
      ksplit = (int)S;
      k64_split = (int)bks;
      n_host = (int)(ceil_div(h, kblock) * S);
      n_hbm = (int)(ceil_div(M - h, kblock) * S);
    }
    // swapped operands (N <= 128, same items): the batch is the MMA's M = 128 side, the item's 128
    // weight rows its N side (umma_swap_kernel). Measured 5-12% faster than the weight-rows-as-M
    // form at the Llama TP8 b64 shapes; 256-row items (one instruction per 256 rows) were slower
    // (4 deeper stages instead of 6: profiles/r01/splitk_sweep.txt)
    if (ksplit > 1 && N <= 128 && M % 4 == 0 && (force_swap || !c.force_path)) swap = N <= 64 ? 2 : 1;  // 2: M = 64
    // (kblock, S) alternatives chasing more weight bytes in flight per SM -- 176..256-row items over
    // 120-141 CTAs -- were measured slower than 128-row items (Llama TP8 b64 step 0.989 vs 0.883 ms,
    // profiles/r02/notes.md): the swapped form is paced per stage by the MMA / commit cycle, not by
    // bytes in flight.
  }
  if (force_swap && !swap) return fail(DAK_EUNSUPPORTED, "dak_linear: swapped tcgen05 form needs N <= 128, M %% 4 == 0 and a split-K workspace");
  const long long rmax_host = ksplit > 1 ? std::min<long long>(h, kblock)
                                         : (n_host ? ceil_div(ceil_div(h, rg), n_host) * rg : 0);
  const long long rmax_hbm = ksplit > 1 ? std::min<long long>(M - h, kblock)
                                        : (n_hbm ? ceil_div(ceil_div(M - h, rg), n_hbm) * rg : 0);
  const long long rmax = std::max(rmax_host, rmax_hbm);
  if (rmax > cap) return fail(DAK_EUNSUPPORTED, "dak_linear: %lld rows per CTA exceed the path capacity %lld (use a smaller kc)", rmax, cap);

  // unroll bucket and the rows one stage must hold (MMA tiles read whole 16-row groups)
  long long rows_alloc;
  int bucket, wm = 1, wk = 1;
  if (path == 1) {
    const int G = kConsumers / (kc / 8);
    bucket = bucket_of(kRptBuckets, 5, ceil_div(rmax, G));
    rows_alloc = ceil_div(rmax, 16) * 16;
  } else if (path == 3) {
    bucket = 1;
    rows_alloc = swap ? ceil_div(rmax, 16) * 16 : ceil_div(rmax, 8) * 8;  // swapped: MMA N % 16 == 0
  } else {
    // warps split K first (the split depends on KC only, so the summation order of a row does
    // not depend on how many rows its CTA owns: bitwise r-invariance); leftover warps split M
    const int KS = kc / 16;
    wk = KS < kConsumerWarps ? KS : kConsumerWarps;
    wm = kConsumerWarps / wk;
    bucket = bucket_of(kMtwBuckets, 7, ceil_div(ceil_div(rmax, 16), wm));
    if (bucket > mtw_max_for(nt)) bucket = -1;
    rows_alloc = (long long)wm * bucket * 16;
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
  if (a->l2_prefetch_bytes > 0) {
    if (!a->l2_prefetch || !aligned16(a->l2_prefetch) || a->l2_prefetch_bytes % 16)
      return fail(DAK_EINVAL, "dak_linear: l2_prefetch must be 16-byte aligned with a multiple-of-16 size");
    p.pf = (const char*)a->l2_prefetch;
    p.pf_bytes = a->l2_prefetch_bytes;
  }
  p.evict_first = c.l2_policy == 0;
  if (p.ldy < M) return fail(DAK_EINVAL, "dak_linear: ldy < M");
  if (pair) {  // groups of G consecutive CTAs, one G-CTA cluster each when W is multicast
    if (path != 3) return fail(DAK_EUNSUPPORTED, "dak_linear: N > 512 needs the tcgen05 path");
    n_host *= G;
    n_hbm *= G;
    p.pair = G;
    p.wmc = c.cluster >= 2 ? 1 : 0;  // cluster >= 2 at N > 512: W multicast across the group
  }
  p.n_host = n_host; p.n_hbm = n_hbm;
  p.wm = wm; p.wk = wk;
  p.rgran = rg;
  if (path == 3) {
    const int cols = (n8 >= 128 ? 1 : 4) * (int)ceil_div(rmax, 128) * n8;  // k-chain accumulators
    p.ksplit = ksplit;
    p.k64_split = k64_split;
    if (ksplit > 1) {
      const size_t need = (size_t)ksplit * N * M * 4;
      if (a->workspace_bytes < (int64_t)need) return fail(DAK_EINVAL, "dak_linear: split-K workspace %lld < %zu", (long long)a->workspace_bytes, need);
      if (!aligned16(a->workspace)) return fail(DAK_EINVAL, "dak_linear: workspace must be 16-byte aligned");
      p.part = (float*)a->workspace;
    }
    p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
    if (swap) p.tmem_cols = kblock <= 32 ? 32 : kblock <= 64 ? 64 : kblock <= 128 ? 128 : 256;  // D[batch][kblock rows], pow2
    p.swap = swap;
    p.kblock = kblock;
  }
  p.mc = mc;
  p.w_stage_bytes = (int)(rows_alloc * kc * 2);
  p.n8 = swap ? (swap == 2 ? 64 : 128) : n8;  // swapped: the batch is the MMA's M side (TMA zero-fills rows >= N)
  p.x_stage_bytes = swap ? p.n8 * 128 : (int)x_stage;  // [kc/64 atoms][n8 rows][64] (x2: gate, up), 128B-swizzled, 1 KB multiple
  p.swiglu = a->x_swiglu ? 1 : 0;
  int ln_bytes = 0;
  if (a->ln_w) {
    if (path == 1) return fail(DAK_EUNSUPPORTED, "dak_linear: fused pre-norm needs a tensor-core path");
    if (K > 8192) return fail(DAK_EUNSUPPORTED, "dak_linear: fused pre-norm keeps LN weights resident: K <= 8192");
    ln_bytes = (int)ceil_div((a->ln_b ? 4 : 2) * K, 128) * 128;
    if (!a->ln_stats || a->ln_parts <= 0) return fail(DAK_EINVAL, "dak_linear: ln_w set but ln_stats / ln_parts missing");
    if (!aligned16(a->ln_w) || !aligned16(a->ln_b) || !aligned16(a->ln_stats))
      return fail(DAK_EINVAL, "dak_linear: ln_w / ln_b / ln_stats must be 16-byte aligned");
    if (a->ln_rms && a->ln_b) return fail(DAK_EINVAL, "dak_linear: RMSNorm takes no bias");
    p.ln_w = (const __nv_bfloat16*)a->ln_w;
    p.ln_b = (const __nv_bfloat16*)a->ln_b;
    p.ln_stats = a->ln_stats;
    p.ln_parts = a->ln_parts;
    p.ln_eps = a->ln_eps;
    p.ln_rms = a->ln_rms ? 1 : 0;
  }
  if (a->stats_out && !aligned16(a->stats_out)) return fail(DAK_EINVAL, "dak_linear: stats_out must be 16-byte aligned");
  p.stats_out = a->stats_out;
  const int W2 = (path == 1 && kc / 8 > 32) ? kc / 8 / 32 : 1;
  // MMA path: one partial slot per k-warp when they fit in 48 KB (one barrier), else serial rounds
  p.red_slots = (path == 2 && wk > 1 && (long long)wk * rmax * N * 4 <= 48 * 1024) ? wk : 1;
  // tcgen05 path: no SMEM results; 16 KB of slack for the M = 128 tile reads past a slot
  const int res_bytes = path == 3 ? 16 * 1024 : (int)(ceil_div((long long)std::max(W2, p.red_slots) * rmax * N * 4, 128) * 128);
  const int per_stage = p.w_stage_bytes + p.x_stage_bytes;
  // SMEM (from a 1024-aligned base; +1 KB for the alignment pad): [1 KB barriers + LN stats]
  // [stages x W span][stages x x box][LN weight, bias][fp32 results]
  int max_stages = (kSmemBudget - 2048 - ln_bytes - res_bytes) / per_stage;
  if (max_stages < 2) return fail(DAK_EUNSUPPORTED, "dak_linear: stage of %d B does not fit twice in SMEM (use a smaller kc)", per_stage);
  max_stages = std::min(max_stages, kMaxStages);
  int stages = c.stages > 0 ? std::min(c.stages, max_stages) : max_stages;
  if (stages < 2) stages = 2;
  p.stages = stages;
  // host CTAs own fewer rows than HBM CTAs: their slots are packed densely inside the same W ring
  // region, so the host ring is deeper (more bytes in flight over the link, which needs >= ~256 KB
  // to saturate; profiles/r01/calib_loadpath.jsonl). MMA tiles read whole rows_alloc groups past a
  // slot's end: that over-read stays inside the region.
  p.w_stage_host = p.w_stage_bytes;
  p.stages_host = stages;
  if (n_host > 0 && !swap) {  // (the swapped kernel uses one slot size for both tiers)
    const long long rh = std::min<long long>(rows_alloc, ceil_div(rmax_host, 16) * 16);
    const long long ws_h = rh * kc * 2;
    const long long over = (rows_alloc - rh) * kc * 2;
    const long long region = (long long)stages * p.w_stage_bytes;
    int sh = (int)std::min<long long>(kMaxStages, (region - over) / ws_h);
    // the x ring needs as many slots: shrink until the whole layout still fits
    while (sh > stages && 1024 + region + (long long)sh * p.x_stage_bytes + ln_bytes + res_bytes + 1024 > kSmemBudget) --sh;
    if (sh > stages) {
      p.w_stage_host = (int)ws_h;
      p.stages_host = sh;
    }
  }
  // congestion window: in-flight host stages per host CTA. With congestion control the
  // window is the smallest that keeps ~256 KB in flight on the link (calibrated saturation point);
  // without it every host ring slot may be in flight.
  // Split-K plans have one host CTA per (row block, K split) item: with congestion control the
  // host_gate semaphore lets at most n_cta_host (default 2) of them stream at once, and the window
  // is sized for that many.
  p.host_gate = 0;
  if (ksplit > 1 && n_host > 0 && c.congestion_control) {
    const int cap_items = c.n_cta_host > 0 ? c.n_cta_host : 2;
    if (n_host > cap_items) p.host_gate = cap_items;
  }
  const int n_stream_host = p.host_gate > 0 ? p.host_gate : n_host;
  int window = p.stages_host;
  if (n_host > 0) {
    if (c.window > 0) window = std::min(c.window, p.stages_host);
    else if (c.congestion_control) {
      const long long hstage = std::max<long long>(1, rmax_host * kc * 2);
      const long long budget = c.host_inflight_kb > 0 ? (long long)c.host_inflight_kb * 1024 : 256 * 1024;  // dak_calibrate
      window = (int)std::min<long long>(p.stages_host, std::max<long long>(1, ceil_div(budget, hstage * n_stream_host)));
    }
  }
  p.window = std::max(1, window);
  const int x_slots = std::max(stages, p.stages_host);
  p.off_x = 1024 + stages * p.w_stage_bytes;
  p.off_ln = p.off_x + x_slots * p.x_stage_bytes;
  p.res_offset = p.off_ln + ln_bytes;

  // CTA-pair GEMM (umma_pair_kernel): the compute-bound large-N regime. Auto when every row is in
  // HBM (h == 0) and N > 256 for a plain GEMM: 7168^2 at N = 512 / 1024 / 2048 / 4096 runs 1.12 /
  // 1.43 / 1.41 / 1.54x faster than the one-CTA forms (tools/pair_bench.py, ~1.06 PFLOP/s); at
  // N = 256 the two tie. A host tier keeps the split paths (their weight-tile multicast groups cross
  // the link once per tile, Table 1); cluster >= 2 asks for them explicitly.
  const bool plain = !a->ln_w && !a->x_swiglu && !a->stats_out;
  if (force_pair && !(kc == 64 && plain))
    return fail(DAK_EUNSUPPORTED, "dak_linear: the CTA-pair GEMM needs kc = 64 and a plain GEMM (no pre-norm / SwiGLU / statistics)");
  if (path == 3 && kc == 64 && plain &&
      (force_pair || (!c.force_path && N > 256 && h == 0 && c.cluster <= 1 && c.n_cta_hbm <= 0))) {
    int nsm = 0;
    dak_status st2 = device_sms(&nsm);
    if (st2 != DAK_OK) return st2;
    const int NB = N > 256 ? 512 : 256;  // batch columns per pair tile (two N = 256 instructions above 256)
    const long long HP = ceil_div(h, 256), GP = ceil_div(M - h, 256), CT = ceil_div(N, NB);
    const long long base = (HP + GP) * CT;  // pair items without a K split
    const long long C = K / 64;
    // K splits from (M, N, K, SM count) only (never h: the summation order of a row does not depend
    // on the tier split): as many as keep every pair item in one wave; fp32 partials need workspace
    long long S = a->workspace ? std::max<long long>(1, std::min<long long>(std::min<long long>(16, C), (nsm / 2) / base)) : 1;
    long long kps = ceil_div(C, S);
    S = ceil_div(C, kps);
    if (S > 1) {
      const size_t need = (size_t)S * N * M * 4;
      if (a->workspace_bytes < (int64_t)need)
        return fail(DAK_EINVAL, "dak_linear: split-K workspace %lld < %zu", (long long)a->workspace_bytes, need);
      if (!aligned16(a->workspace)) return fail(DAK_EINVAL, "dak_linear: workspace must be 16-byte aligned");
      p.part = (float*)a->workspace;
    }
    const int per_stage = 16384 * (1 + NB / 256);
    p.stages = std::min(kMaxStages, (kSmemBudget - 2048) / per_stage);
    if (c.stages > 0) p.stages = std::max(2, std::min(p.stages, c.stages));
    p.pair2 = NB;
    p.p2_hp = (int)HP;
    p.p2_ct = (int)CT;
    p.ksplit = (int)S;
    p.k64_split = (int)kps;
    p.n8 = 128;  // x TMA box: 128 rows (this CTA's half of a 256-column block)
    p.x_stage_bytes = 16384 * (NB / 256);
    p.swap = 0;
    p.pair = 1;
    p.wmc = 0;
    p.mc = 1;
    p.host_gate = 0;
    p.n_host = (int)(2 * HP * CT * S);
    p.n_hbm = (int)(2 * GP * CT * S);
    p.kblock = 256;
    out->p = p;
    out->path = 3;
    out->nn = 0;
    out->bucket = 0;
    out->grid = p.n_host + p.n_hbm;
    out->smem = 1024 + p.stages * per_stage + 1024;
    out->rmax_host = HP ? std::min<long long>(h, 128) : 0;
    out->rmax_hbm = GP ? std::min<long long>(M - h, 128) : 0;
    return DAK_OK;
  }
  out->p = p;
  out->path = path;
  out->nn = path == 1 ? N : nt_eff;
  out->bucket = bucket;
  out->grid = n_host + n_hbm;
  out->smem = p.res_offset + res_bytes + 1024;
  out->rmax_host = rmax_host;
  out->rmax_hbm = rmax_hbm;
  return DAK_OK;
}

// x [N, K] bf16 as a 3-D tensor (64 elements, N rows, K/64 atoms): one box [64, n8, kc/64] per
// stage, 128-byte swizzle, rows >= N zero-filled by the TMA unit.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static dak_status encode_xmap(Params* p) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    DAK_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) return fail(DAK_ECUDA, "dak_linear: cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)f;
  }
  const long long ldx = p->swiglu ? 2 * p->K : p->K;  // [gate | up] rows are 2K wide
  const cuuint64_t dims[3] = {64, (cuuint64_t)p->N, (cuuint64_t)(ldx / 64)};
  const cuuint64_t strides[2] = {(cuuint64_t)ldx * 2, 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)(p->n8 > 256 ? 256 : p->n8), (cuuint32_t)(p->kc / 64)};  // TMA box <= 256 rows
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&p->xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)p->x, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DAK_ECUDA, "dak_linear: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DAK_OK;
}
// CTA-pair GEMM weight maps: a tier's DAK-KC block [K/64 chunks][R rows][64 elements] (rows stored
// 128B-swizzled by row & 7) as (64 elements, R rows, K/64 chunks), box (64, 128, 1), no swizzle:
// a box of 128 rows starting at a multiple of 128 lands as the canonical SWIZZLE_128B operand
static dak_status encode_wmaps(Params* p) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    DAK_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) return fail(DAK_ECUDA, "dak_linear: cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)f;
  }
  const long long R[2] = {p->M - p->h, p->h};
  const char* base[2] = {p->w_hbm, p->w_host};
  for (int t = 0; t < 2; ++t) {
    if (R[t] <= 0 || !base[t]) continue;
    const cuuint64_t dims[3] = {64, (cuuint64_t)R[t], (cuuint64_t)(p->K / 64)};
    const cuuint64_t strides[2] = {128, (cuuint64_t)R[t] * 128};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(&p->wmap[t], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)base[t], dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(DAK_ECUDA, "dak_linear: weight tensor map failed (%d)", (int)r);
  }
  return DAK_OK;
}

template <int PATH, int NN, int B, int XF>
static dak_status launch_t(const Plan& pl, cudaStream_t stream, int pdl) {
  auto kern = split_linear_kernel<PATH, NN, B, XF>;
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
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = pl.p.mc;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pl.p.mc > 1 ? 2 : 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, pl.p));
  return DAK_OK;
}

template <int NN>
static dak_status launch_fma(const Plan& pl, cudaStream_t s, int pdl) {
  switch (pl.bucket) {
    case 1: return launch_t<1, NN, 1, 0>(pl, s, pdl);
    case 2: return launch_t<1, NN, 2, 0>(pl, s, pdl);
    case 4: return launch_t<1, NN, 4, 0>(pl, s, pdl);
    case 8: return launch_t<1, NN, 8, 0>(pl, s, pdl);
    case 16: return launch_t<1, NN, 16, 0>(pl, s, pdl);
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no FMA kernel instance for bucket %d", pl.bucket);
}

template <int NT, int XF>
static dak_status launch_mma(const Plan& pl, cudaStream_t s, int pdl) {
  switch (pl.bucket) {
    case 1: return launch_t<2, NT, 1, XF>(pl, s, pdl);
    case 2: return launch_t<2, NT, 2, XF>(pl, s, pdl);
    case 3: return launch_t<2, NT, 3, XF>(pl, s, pdl);
    case 4: return launch_t<2, NT, 4, XF>(pl, s, pdl);
  }
  if constexpr (NT <= 4) {
    switch (pl.bucket) {
      case 6: return launch_t<2, NT, 6, XF>(pl, s, pdl);
      case 8: return launch_t<2, NT, 8, XF>(pl, s, pdl);
    }
  }
  if constexpr (NT <= 2) {
    if (pl.bucket == 12) return launch_t<2, NT, 12, XF>(pl, s, pdl);
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no MMA kernel instance for bucket %d / %d n8 tiles", pl.bucket, NT);
}

template <int NT>
static dak_status launch_mma_xf(const Plan& pl, cudaStream_t s, int pdl) {
  if (pl.p.ln_w) return launch_mma<NT, 1>(pl, s, pdl);
  if (pl.p.swiglu) return launch_mma<NT, 2>(pl, s, pdl);
  return launch_mma<NT, 0>(pl, s, pdl);
}

#if DAK_LINEAR_PART == 6
// ================================================================================================
// CTA-pair tcgen05 GEMM for the compute-bound large-N regime:
// a cluster of two CTAs on one TPC computes a tile of 256 weight rows x 256 NI batch columns with
// ONE stream of tcgen05.mma.cta_group::2 instructions (M = 256, N = 256, K = 16) issued by the
// leader CTA. Each CTA stages ITS 128 weight rows (A) and ITS half of every 256-column x block (B)
// at the same shared-memory offsets; the tensor cores read both CTAs' operands and each CTA's TMEM
// receives its 128 rows of D. Measured (tools/umma2_micro.cu): 128 cycles per M = 256 x N = 256 x
// K = 16 instruction = the full dense rate per SM, where the one-CTA form pays >= 100 cycles per
// M = 128 instruction; and each SM ingests half the x bytes per FLOP (the bound of the one-CTA form
// at large N: profiles/r02/s3/f1_large_n_ncu.txt).
// Items: (tier row pair, batch-column tile, K split), host-tier pairs first (a CTA pair
// reads one tier); the splits S are fixed by (M, K, N) -- fp32 partials reduced by
// splitk_reduce_kernel in split order, as the split-K path. Both CTAs' W and x loads are tensor
// TMAs with .cta_group::2 completing on the LEADER's stage barrier (which expects the pair's bytes);
// a first version relayed the peer's arrival through a remote mbarrier arrive and ran at ~0.9
// PFLOP/s instead of ~1.06. Stage release and accumulator completion are tcgen05.commit multicasts
// to both CTAs.
constexpr int kPairThreads = 192;  // warp 0 producer, warp 1 MMA issuer (leader) / relay (peer), 2-5 epilogue

__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   su32(bar)),
               "h"((uint16_t)3)
               : "memory");
}
// 3-D tensor TMA into this CTA's shared memory completing on a barrier of the CTA pair (shared::cluster
// address, e.g. the leader's via mapa)
__device__ __forceinline__ void tma_3d_2sm(void* dst, uint64_t tmap, int c0, int c1, int c2, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}

template <int NI>  // 256-column MMA instructions per K step: pair tile = 256 rows x 256 NI columns
__global__ void __launch_bounds__(kPairThreads, 1) umma_pair_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [kMaxStages] leader: the pair's stage landed
  uint64_t* empty = full + kMaxStages;                  // [kMaxStages] the pair's MMAs read the stage
  uint64_t* done = empty + kMaxStages;                  // accumulators complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 512);
  const uint32_t rank = cta_rank_in_cluster();
  const int item = (int)(blockIdx.x >> 1);
  const int S = p.ksplit > 1 ? p.ksplit : 1;
  const int CT = p.p2_ct;
  const int host_items = p.p2_hp * CT * S;
  const bool host = item < host_items;
  const int it = host ? item : item - host_items;
  const int ks = it % S;
  const int ct = (it / S) % CT;
  const int rp = it / (S * CT);
  const long long R_tier = host ? p.h : p.M - p.h;
  const long long rb = (long long)rp * 256 + 128 * (long long)rank;  // this CTA's first row in its tier
  const int R = (int)max(0LL, min(128LL, R_tier - rb));
  const char* wsrc = host ? p.w_host : p.w_hbm;
  const long long chunk_stride = R_tier * 128;
  const int C = (int)(p.K / 64);
  const int kbeg = ks * p.k64_split;
  const int kend = min(C, kbeg + p.k64_split);
  const int nch = kend - kbeg;
  const int slots = p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kW = 16384, kX = 16384 * NI;  // per-stage bytes: 128 rows x 64 K, NI x 128 x rows x 64 K
  unsigned char* wring = smem + 1024;
  unsigned char* xring = smem + 1024 + (size_t)slots * kW;
  const int col0 = ct * 256 * NI;  // the tile's first batch column

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(256u * NI)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM exist before any remote arrive / MMA
  tc_fence_after();
  if (threadIdx.x == 0) tstamp(p.trace, 0);
  grid_dep_launch();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0 && nch > 0) {  // producer: this CTA's W rows + its halves of the x blocks per K chunk
      // both CTAs' loads complete on the LEADER's full barrier (.cta_group::2), which expects the
      // pair's bytes; rows past the tier are zero-filled by the tensor map
      const uint64_t xmap = reinterpret_cast<uint64_t>(&p.xmap);
      const uint64_t wmap = reinterpret_cast<uint64_t>(&p.wmap[host ? 1 : 0]);
      asm volatile("prefetch.tensormap [%0];" ::"l"(xmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(wmap) : "memory");
      const int pro = min(slots, nch);
      auto lead_bar = [&](int slot) {
        uint32_t r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(&full[slot])), "r"(0));
        return r;
      };
      auto load_w = [&](int slot, int i) {
        if (rank == 0) mbar_expect_tx(&full[slot], 2u * (kW + kX));
        tma_3d_2sm(wring + (size_t)slot * kW, wmap, 0, (int)rb, kbeg + i, lead_bar(slot));
      };
      auto load_x = [&](int slot, int i) {
#pragma unroll
        for (int j = 0; j < NI; ++j)
          tma_3d_2sm(xring + (size_t)slot * kX + j * 16384, xmap, 0, col0 + 256 * j + 128 * (int)rank, kbeg + i,
                     lead_bar(slot));
      };
      for (int i = 0; i < pro; ++i) load_w(i, i);  // weights do not depend on the previous kernel
      grid_dep_wait();  // x is produced by the previous kernel
      tstamp(p.trace, 1);
      for (int i = 0; i < pro; ++i) load_x(i, i);
      int s = pro == slots ? 0 : pro;
      uint32_t ph = pro == slots ? 1u : 0u;
      for (int i = pro; i < nch; ++i) {
        mbar_spin(&empty[s], ph ^ 1u);
        load_w(s, i);
        load_x(s, i);
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // MMA issuer: the whole warp walks the ring, one elected lane issues
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      const uint32_t wr = su32(wring), xr = su32(xring);
      uint32_t leader;
      asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nch; ++i) {
        mbar_spin(&full[s], ph);  // both CTAs' operands of stage s landed
        tc_fence_after();
        if (leader) {
          const uint32_t ws = wr + (uint32_t)s * kW, xs = xr + (uint32_t)s * kX;
#pragma unroll
          for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma2_bf16(tmem + 256u * j, umma_desc_sw128(ws + k * 32), umma_desc_sw128(xs + j * 16384 + k * 32), idesc,
                         (i | k) != 0);
          umma2_commit_both(&empty[s]);  // both CTAs may refill slot s once these MMAs have read it
        }
        __syncwarp();
        if (++s == slots) { s = 0; ph ^= 1u; }
      }
      if (leader) umma2_commit_both(done);
      __syncwarp();
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. = rows of this CTA's 128
    if (threadIdx.x == 64) {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(done)), "r"(0u) : "memory");
        if (!ok) __nanosleep(256);
      }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    tc_fence_after();
    grid_dep_wait();  // residual / y may belong to the previous kernel
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const long long m = (host ? 0 : p.h) + rb + r;
    const bool ok = r < R && nch > 0;
    const float bias = (ok && p.bias && S == 1) ? __bfloat162float(p.bias[m]) : 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < 256 * NI; c0 += 8) {
      uint32_t v[8];
      tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!ok) continue;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int n = col0 + c0 + e;
        if (n >= p.N) continue;
        const float acc = __uint_as_float(v[e]);
        if (S > 1) {  // raw fp32 partial; bias / act / residual in splitk_reduce_kernel
          p.part[((size_t)ks * p.N + n) * p.M + m] = acc;
        } else {
          float o = acc + bias;
          if (p.act == DAK_ACT_RELU) o = fmaxf(o, 0.f);
          if (p.residual) o += __bfloat162float(p.residual[(long long)n * p.ldy + m]);
          p.y[(long long)n * p.ldy + m] = __float2bfloat16_rn(o);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves while the pair's MMAs / remote arrives may still target it
  if (threadIdx.x == 32 && p.trace) tstamp(p.trace, 3);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u * NI) : "memory");
  }
}

template <int NI>
static dak_status launch_pair_t(const Plan& pl, cudaStream_t stream, int pdl) {
  auto kern = umma_pair_kernel<NI>;
  static int smem_set = 0;
  if (!smem_set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    smem_set = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, pl.p));
  return DAK_OK;
}
dak_status launch_part_pair(const Plan& pl, cudaStream_t s, int pdl) {
  return pl.p.pair2 > 256 ? launch_pair_t<2>(pl, s, pdl) : launch_pair_t<1>(pl, s, pdl);
}
#endif

// The kernel instances are spread over several translation units (this file compiled with
// DAK_LINEAR_PART = 0..4, see build.py) so they compile in parallel; part 0 holds the host code.
dak_status launch_part_fma(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_nt1(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_nt2(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_nt4(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_nt8(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_umma(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_swap(const Plan& pl, cudaStream_t s, int pdl);
dak_status launch_part_pair(const Plan& pl, cudaStream_t s, int pdl);
#if DAK_LINEAR_PART == 0
dak_status launch_part_fma(const Plan& pl, cudaStream_t s, int pdl) {
  switch (pl.nn) {
    case 1: return launch_fma<1>(pl, s, pdl);
    case 2: return launch_fma<2>(pl, s, pdl);
    case 3: return launch_fma<3>(pl, s, pdl);
    case 4: return launch_fma<4>(pl, s, pdl);
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no FMA kernel instance for N = %d", pl.nn);
}
#elif DAK_LINEAR_PART == 1
dak_status launch_part_nt1(const Plan& pl, cudaStream_t s, int pdl) { return launch_mma_xf<1>(pl, s, pdl); }
#elif DAK_LINEAR_PART == 2
dak_status launch_part_nt2(const Plan& pl, cudaStream_t s, int pdl) { return launch_mma_xf<2>(pl, s, pdl); }
#elif DAK_LINEAR_PART == 3
dak_status launch_part_nt4(const Plan& pl, cudaStream_t s, int pdl) { return launch_mma_xf<4>(pl, s, pdl); }
#elif DAK_LINEAR_PART == 4
dak_status launch_part_nt8(const Plan& pl, cudaStream_t s, int pdl) { return launch_mma_xf<8>(pl, s, pdl); }
#elif DAK_LINEAR_PART == 5
template <int NT, int XF>
static dak_status launch_umma_t(const Plan& pl, cudaStream_t stream, int pdl) {
  auto kern = umma_linear_kernel<NT, XF>;
  static int smem_set = 0;
  if (!smem_set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    smem_set = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;  // W multicast groups: one G-CTA cluster per group
  attr[1].val.clusterDim.x = pl.p.pair > 1 && pl.p.wmc ? pl.p.pair : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, pl.p));
  return DAK_OK;
}
template <int NT>
static dak_status launch_umma_xf(const Plan& pl, cudaStream_t s, int pdl) {
  if (pl.p.ln_w) return launch_umma_t<NT, 1>(pl, s, pdl);
  if (pl.p.swiglu) return launch_umma_t<NT, 2>(pl, s, pdl);
  return launch_umma_t<NT, 0>(pl, s, pdl);
}
dak_status launch_part_swap(const Plan& pl, cudaStream_t stream, int pdl) {
  static int smem_set = 0;
  if (!smem_set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(umma_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
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
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, umma_swap_kernel, pl.p));
  return DAK_OK;
}
dak_status launch_part_umma(const Plan& pl, cudaStream_t s, int pdl) {
  switch (pl.nn) {
    case 2: return launch_umma_xf<2>(pl, s, pdl);
    case 4: return launch_umma_xf<4>(pl, s, pdl);
    case 8: return launch_umma_xf<8>(pl, s, pdl);
    case 16: return launch_umma_xf<16>(pl, s, pdl);
    case 32: return launch_umma_xf<32>(pl, s, pdl);
    case 64: return launch_umma_t<64, 0>(pl, s, pdl);  // N 257..512: plain GEMM only
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no tcgen05 kernel instance for %d n8 tiles", pl.nn);
}
#endif

#if DAK_LINEAR_PART == 0
static dak_status launch(const Plan& pl, cudaStream_t s, int pdl) {
  if (pl.grid == 0) return DAK_OK;
  if (pl.path == 1) return launch_part_fma(pl, s, pdl);
  if (pl.path == 3) return pl.p.pair2 ? launch_part_pair(pl, s, pdl) : pl.p.swap ? launch_part_swap(pl, s, pdl) : launch_part_umma(pl, s, pdl);
  switch (pl.nn) {
    case 1: return launch_part_nt1(pl, s, pdl);
    case 2: return launch_part_nt2(pl, s, pdl);
    case 4: return launch_part_nt4(pl, s, pdl);
    case 8: return launch_part_nt8(pl, s, pdl);
  }
  return fail(DAK_EUNSUPPORTED, "dak_linear: no kernel instance for path %d / %d", pl.path, pl.nn);
}
#endif

}  // namespace lin
}  // namespace dak

#if DAK_LINEAR_PART == 0
using namespace dak;

static inline long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }

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

int32_t dak_linear_choose_kc(int64_t rows_per_cta, int64_t K) {
  if (K % 256 == 0 && rows_per_cta <= 96) return 256;
  if (K % 128 == 0 && rows_per_cta <= 192) return 128;
  return 64;
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
  info->cluster = pl.p.mc;
  info->ksplit = pl.path == 3 && pl.p.ksplit > 1 ? pl.p.ksplit : 1;
  info->host_gate = pl.p.host_gate;
  info->kblock = pl.path == 3 && pl.p.ksplit > 1 ? pl.p.kblock : 0;
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
  long long rb, re;
  if (pl.p.pair2) {  // CTA-pair GEMM: CTA = (pair item, rank); item = (row pair, column tile, K split)
    const long long item = j / 2, rank = j % 2;
    const long long rp = item / ((long long)pl.p.p2_ct * std::max(1, pl.p.ksplit));
    rb = std::min<long long>(R, rp * 256 + 128 * rank);
    re = std::min<long long>(R, rb + 128);
  } else if (pl.path == 3 && pl.p.ksplit > 1) {  // split-K: CTA = (row block of kblock rows, K split) item
    rb = std::min<long long>(R, (j / pl.p.ksplit) * pl.p.kblock);
    re = std::min<long long>(R, rb + pl.p.kblock);
  } else if (pl.p.pair > 1) {  // N > 512: groups of `pair` CTAs share one row range
    lin::tier_rows(R, j / pl.p.pair, n / pl.p.pair, pl.p.rgran, &rb, &re);
  } else {
    lin::tier_rows(R, j, n, pl.p.rgran, &rb, &re);
  }
  *tier = host ? 1 : 0;
  *row_begin = off + rb;
  *row_end = off + re;
  return DAK_OK;
}

dak_status dak_linear(const dak_linear_args* args, dak_stream_t stream) {
  return dak::linear_enqueue(args, stream, false, nullptr);
}

}  // extern "C"

dak_status dak::linear_enqueue(const dak_linear_args* args, void* stream, bool defer_reduce, int* ksplit_out) {
  lin::Plan pl;
  dak_status st = lin::make_plan(args, &pl);
  if (st != DAK_OK) return st;
  if (pl.grid && !(pl.p.y)) return fail(DAK_EINVAL, "dak_linear: y NULL");
  if (pl.grid && (st = lin::encode_xmap(&pl.p)) != DAK_OK) return st;
  if (pl.grid && pl.p.pair2 && (st = lin::encode_wmaps(&pl.p)) != DAK_OK) return st;
  pl.p.trace = trace_slot(DAK_KIND_LINEAR, args->M, args->K, pl.grid);
  if ((st = lin::launch(pl, (cudaStream_t)stream, args->cfg.pdl)) != DAK_OK) return st;
  const int S = pl.path == 3 && pl.p.ksplit > 1 ? pl.p.ksplit : 1;
  if (ksplit_out) *ksplit_out = S;
  if (S > 1 && !defer_reduce) {
    const int vec = args->M % 4 == 0 && pl.p.ldy % 4 == 0 && ((uintptr_t)pl.p.y & 7) == 0 &&
                    ((uintptr_t)pl.p.residual & 7) == 0 && ((uintptr_t)pl.p.bias & 7) == 0;
    const long long per_row = vec ? args->M / 4 : args->M;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = args->cfg.pdl ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    const long long gx = std::min<long long>(ceil_div_ll(per_row, 256), 64);
    cfg.gridDim = dim3((unsigned)gx, (unsigned)args->N);
    cfg.blockDim = dim3(256);
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, lin::splitk_reduce_kernel, (const float*)pl.p.part, pl.p.ksplit, (int)args->N,
                                    (long long)args->M, pl.p.bias, pl.p.act, pl.p.residual, pl.p.y, pl.p.ldy, vec,
                                    trace_slot(DAK_KIND_REDUCE, args->M, pl.p.ksplit, (int)(cfg.gridDim.x * cfg.gridDim.y))));
  }
  return DAK_OK;
}

extern "C" {

size_t dak_linear_workspace_size(const dak_linear_args* args) {
  if (!args) return 0;
  dak_linear_args a = *args;
  a.workspace = (void*)16;  // probe: would the plan split K?
  a.workspace_bytes = INT64_MAX;
  lin::Plan pl;
  if (lin::make_plan(&a, &pl) != DAK_OK || pl.p.ksplit <= 1) return 0;
  return (size_t)pl.p.ksplit * a.N * a.M * 4;
}

}  // extern "C"

#endif  // DAK_LINEAR_PART == 0
