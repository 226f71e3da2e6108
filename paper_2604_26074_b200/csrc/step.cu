// dak_step — persistent decode-step kernel for sm_100a (PAPER §3.1, §4).
//
// One launch executes a whole decode step described by an op table (embed, LayerNorm, split
// linear, split paged attention, split-KV combine). Grid = one CTA per SM, all co-resident.
// Each CTA runs three roles over the same op sequence:
//   warp 0 (stream producer)  : streams this CTA's weight rows / KV pages of every op, back to back,
//                               into an SMEM ring with 1-D bulk copies (TMA engine) from HBM or
//                               pinned host memory (each CTA one tier per op; host stages
//                               capped by the congestion window). Weights never depend on
//                               activations, so the stream runs ahead across op boundaries: the
//                               memory pipe does not drain between ops (no launch ramp / tail).
//   warp 1 (x producer)       : waits (gpu-scope acquire on a completion counter) for the op whose
//                               output this op reads, then bulk-copies the x chunk (or q rows) of
//                               every stage next to the weights.
//   warps 2..9 (consumers)    : mma.sync m16n8k16 on the staged tiles (same math and reduction
//                               order as dak_linear / dak_attention), epilogues (bias, ReLU,
//                               residual, LN statistics, fused KV append), LN / embed / combine
//                               work, then a release-increment of the op's completion counter.
// Counters are reset by the last CTA to finish, so the launch is replayable (CUDA graphs).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.h"
#include "ptx.cuh"

namespace dak {
namespace step {
using namespace dak::ptx;

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = 64 + kConsumers;
constexpr int kNB = 12;  // barrier pairs (max stages in flight)
constexpr int kHeader = 2048;        // barriers, LN statistics, per-role op descriptor copies
constexpr int kAlign = 1024;         // ring stage placement granule (bytes)
constexpr int kL1Reserve = 16 * 1024;  // left to L1 (spills, stack, op-table misses)
constexpr int kD = 128;
constexpr int kGmax = 8;
constexpr int kQPitch = kD * 2 + 16;
constexpr int kMtwMax = 12;
constexpr int kSmemBudget = 227 * 1024;
constexpr uint32_t kHostBit = 0x80000000u;
constexpr int kScratch = kConsumerWarps * (kGmax * kD + 2 * kGmax) * 4;  // attention merge / linear reduce

struct alignas(16) Op {
  int type, dep, n_host, n_hbm;
  // linear
  const char* w_host;
  const char* w_hbm;
  long long M, K, h;
  int kc, act, rb_rows, window;
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  float* stats_out;
  long long kv_row0;  // first row appended to the KV cache (-1: no append)
  int kv_kind;        // 1: k rows, 2: v rows, 3: fused [k; v] rows
  long long ldy;      // row stride of y and residual
  // embed / layernorm
  const float* stats_in;
  const __nv_bfloat16* ln_w;
  const __nv_bfloat16* ln_b;
  float eps;
  int cols;
  const int* tokens;
  const int* positions;
  const __nv_bfloat16* tok_emb;
  const __nv_bfloat16* pos_emb;
  int pos_offset;
  // attention / combine / append
  const __nv_bfloat16* q;
  long long q_stride;
  __nv_bfloat16* out;
  char* k_hbm;
  char* v_hbm;
  char* k_host;
  char* v_host;
  const int* block_table;
  const int* seq_lens;
  int Hq, Hkv, G, page, max_pages, chunk_pages, max_chunks;
  float scale_log2;
  const int* units_host;
  const int* units_hbm;
  int n_units_host, n_units_hbm;
  float* part_o;
  float* part_lse;
};

struct Params {
  const Op* ops;
  int n_ops, N, ring_bytes;
  int* done;      // [n_ops] completion counters
  int* finished;  // CTAs that finished the launch
  int off_scratch;
  unsigned long long* trace;  // optional [n_ops][grid][4] globaltimer stamps (ns)
};

// ---------------------------------------------------------------------------------- helpers
struct LinRole {
  bool active, host;
  long long rb, re, R_tier;
  const char* wsrc;
};
__device__ __forceinline__ LinRole lin_role(const Op& op, int cta) {
  LinRole r;
  r.host = cta < op.n_host;
  const int j = r.host ? cta : cta - op.n_host;
  const int n = r.host ? op.n_host : op.n_hbm;
  r.R_tier = r.host ? op.h : op.M - op.h;
  r.active = j < n && r.R_tier > 0;
  r.rb = r.active ? (long long)j * r.R_tier / n : 0;
  r.re = r.active ? (long long)(j + 1) * r.R_tier / n : 0;
  r.wsrc = r.host ? op.w_host : op.w_hbm;
  return r;
}
struct AttRole {
  bool host;
  int j, n, n_units;
  const int* units;
};
__device__ __forceinline__ AttRole att_role(const Op& op, int cta) {
  AttRole r;
  r.host = cta < op.n_host;
  r.j = r.host ? cta : cta - op.n_host;
  r.n = r.host ? op.n_host : op.n_hbm;
  r.units = r.host ? op.units_host : op.units_hbm;
  r.n_units = (r.host ? op.n_units_host : op.n_units_hbm) * op.Hkv;
  if (r.j >= r.n) r.n_units = 0;
  return r;
}
struct Unit {
  int b, g, c, L, pg0, pg1;
};
__device__ __forceinline__ Unit att_unit(const Op& op, const AttRole& r, int k) {
  Unit u;
  const int pr = r.units[k / op.Hkv];
  u.g = k % op.Hkv;
  u.b = pr / op.max_chunks;
  u.c = pr % op.max_chunks;
  u.L = op.seq_lens[u.b];
  const int npg = (u.L + op.page - 1) / op.page;
  u.pg0 = u.c * op.chunk_pages;
  u.pg1 = min(npg, u.pg0 + op.chunk_pages);
  return u;
}
// Byte-addressed ring: stage i occupies [off, off + sz) of the ring; a stage that does not fit
// before the end wraps to offset 0. Every role walks the same stage sequence, so every role
// computes the same offsets. Barrier pair i % kNB guards stage i.
struct Cur {
  long long i;
  int off, sz;
};
__device__ __forceinline__ void cur_next(Cur& c, int sz, int RB) {
  ++c.i;
  int o = c.off + c.sz;
  if (o + sz > RB) o = 0;
  c.off = o;
  c.sz = sz;
}
__device__ __forceinline__ int lin_stage_w(int R, int kc) { return (R * kc * 2 + kAlign - 1) & ~(kAlign - 1); }
__device__ __forceinline__ int lin_stage_bytes(int R, int kc, int N8) {
  return lin_stage_w(R, kc) + ((N8 * (kc * 2 + 16) + kAlign - 1) & ~(kAlign - 1));
}
__device__ __forceinline__ int att_stage_bytes(int pb) { return 2 * pb + ((kGmax * kQPitch + kAlign - 1) & ~(kAlign - 1)); }

// ---------------------------------------------------------------------------------- MMA stage
template <int NT, int MTW>
__device__ __forceinline__ void mma_stage(float (&acc)[kMtwMax][NT][4], uint32_t ws, uint32_t xs, int kc, int wk,
                                          int WK, int nks, uint32_t a_step, int key, int ahalf) {
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
}

// ---------------------------------------------------------------------------------- kernel
template <int NT>
__global__ void __launch_bounds__(kThreads, 1) step_kernel(const Params P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kNB;
  uint64_t* ready = empty + kNB;  // stream producer -> x producer: stage region is free
  float* s_stat = reinterpret_cast<float*>(ready + kNB);  // [16][2] LN mean / rstd
  unsigned char* ring = smem + kHeader;
  float* scratch = reinterpret_cast<float*>(smem + P.off_scratch);
  const int cta = blockIdx.x, G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RB = P.ring_bytes;
  // per-role SMEM copy of the current op descriptor (the table lives in global memory; with the
  // ring taking most of the unified L1/SMEM, field reads would otherwise go to L2)
  Op* const sop = reinterpret_cast<Op*>(smem + 512 + 512 * (warp == 0 ? 0 : warp == 1 ? 1 : 2));
  unsigned long long* const TR = P.trace;
#define DAK_TRACE(oi, k) \
  do {                    \
    if (TR) TR[((long long)(oi) * G + cta) * 4 + (k)] = gtime(); \
  } while (0)
  const int N = P.N;
  const int N8 = (N + 7) & ~7;

  if (threadIdx.x == 0) {
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&full[b], 2);  // stream producer (expect_tx) + x producer (expect_tx / arrive)
      mbar_init(&empty[b], kConsumerWarps);
      mbar_init(&ready[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ======================================================== stream producer (weights / KV pages)
    if (lane == 0) {
      Cur cur{-1, 0, 0};
      long long oldest = 0;    // oldest stage not yet known to be consumed
      // byte regions of the in-flight stages (index i % kNB), in SMEM (not local memory)
      int* reg_lo = reinterpret_cast<int*>(smem + 416);
      int* reg_hi = reg_lo + kNB;
      // place stage i: wait until its ring region and its barrier pair are free (stages are
      // consumed in order, so waiting on stage j implies every earlier stage is consumed)
      auto acquire = [&](int sz, int win) {
        cur_next(cur, sz, RB);
        const long long i = cur.i;
        while (oldest < i && (i - oldest >= kNB || i - oldest >= win)) {
          mbar_wait(&empty[oldest % kNB], (uint32_t)((oldest / kNB) & 1));
          ++oldest;
        }
        for (long long j = oldest; j < i; ++j) {
          const int b = (int)(j % kNB);
          if (reg_lo[b] < cur.off + sz && cur.off < reg_hi[b]) {
            mbar_wait(&empty[b], (uint32_t)((j / kNB) & 1));
            oldest = j + 1;
          }
        }
        const int b = (int)(i % kNB);
        reg_lo[b] = cur.off;
        reg_hi[b] = cur.off + sz;
        mbar_arrive(&ready[b]);
        return b;
      };
      for (int oi = 0; oi < P.n_ops; ++oi) {
        {
          const int4* src = reinterpret_cast<const int4*>(P.ops + oi);
          int4* dst = reinterpret_cast<int4*>(sop);
          for (int k = 0; k < (int)(sizeof(Op) / 16); ++k) dst[k] = src[k];
        }
        const Op& op = *sop;
        if (op.type == DAK_STEP_LINEAR) {
          const LinRole r = lin_role(op, cta);
          if (!r.active) continue;
          const int nch = (int)(op.K / op.kc);
          const long long cstride = r.R_tier * op.kc * 2;
          const int win = r.host ? op.window : kNB;
          for (long long r0 = r.rb; r0 < r.re; r0 += op.rb_rows) {
            const int R = (int)min((long long)op.rb_rows, r.re - r0);
            const uint32_t wb = (uint32_t)R * op.kc * 2;
            const int sz = lin_stage_bytes(R, op.kc, N8);
            const char* src = r.wsrc + r0 * op.kc * 2;
            for (int c = 0; c < nch; ++c) {
              const int b = acquire(sz, win);
              mbar_expect_tx(&full[b], wb);
              bulk_g2s(ring + cur.off, src + (long long)c * cstride, wb, &full[b]);
            }
          }
        } else if (op.type == DAK_STEP_ATTENTION) {
          const AttRole r = att_role(op, cta);
          if (r.n_units == 0) continue;
          spin_until_geq(&P.done[op.dep], G);  // the new token's K/V rows come from the k/v epilogues
          DAK_TRACE(oi, 0);
          fence_proxy_async();
          const int pb = op.page * kD * 2;
          const int win = r.host ? op.window : kNB;
          for (int k = r.j; k < r.n_units; k += r.n) {
            const Unit u = att_unit(op, r, k);
            for (int pg = u.pg0; pg < u.pg1; ++pg) {
              const int b = acquire(att_stage_bytes(pb), win);
              const uint32_t e = (uint32_t)op.block_table[(long long)u.b * op.max_pages + pg];
              const long long off = ((long long)(e & ~kHostBit) * op.Hkv + u.g) * pb;
              const bool eh = (e & kHostBit) != 0;
              mbar_expect_tx(&full[b], 2u * pb);
              bulk_g2s(ring + cur.off, (eh ? op.k_host : op.k_hbm) + off, pb, &full[b]);
              bulk_g2s(ring + cur.off + pb, (eh ? op.v_host : op.v_hbm) + off, pb, &full[b]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================================================== x producer (activations, q rows)
    Cur cur{-1, 0, 0};
    for (int oi = 0; oi < P.n_ops; ++oi) {
      __syncwarp();
      for (int k = lane; k < (int)(sizeof(Op) / 16); k += 32)
        reinterpret_cast<int4*>(sop)[k] = reinterpret_cast<const int4*>(P.ops + oi)[k];
      __syncwarp();
      const Op& op = *sop;
      if (op.type == DAK_STEP_LINEAR) {
        const LinRole r = lin_role(op, cta);
        if (!r.active) continue;
        if (lane == 0 && op.dep >= 0) spin_until_geq(&P.done[op.dep], G);
        if (lane == 0) DAK_TRACE(oi, 1);
        __syncwarp();
        fence_proxy_async();
        const int nch = (int)(op.K / op.kc);
        const uint32_t xb = (uint32_t)op.kc * 2;
        const int pitch = op.kc * 2 + 16;
        for (long long r0 = r.rb; r0 < r.re; r0 += op.rb_rows) {
          const int R = (int)min((long long)op.rb_rows, r.re - r0);
          const int sz = lin_stage_bytes(R, op.kc, N8);
          const int xo = lin_stage_w(R, op.kc);
          for (int c = 0; c < nch; ++c) {
            cur_next(cur, sz, RB);
            const int b = (int)(cur.i % kNB);
            if (lane == 0) {
              mbar_wait(&ready[b], (uint32_t)((cur.i / kNB) & 1));
              mbar_expect_tx(&full[b], (uint32_t)N * xb);
            }
            __syncwarp();
            if (lane < N)
              bulk_g2s(ring + cur.off + xo + lane * pitch, op.x + (long long)lane * op.K + (long long)c * op.kc, xb,
                       &full[b]);
          }
        }
      } else if (op.type == DAK_STEP_ATTENTION) {
        const AttRole r = att_role(op, cta);
        if (r.n_units == 0) continue;
        if (lane == 0) spin_until_geq(&P.done[op.dep], G);
        if (lane == 0) DAK_TRACE(oi, 1);
        __syncwarp();
        fence_proxy_async();
        const int pb = op.page * kD * 2;
        for (int k = r.j; k < r.n_units; k += r.n) {
          const Unit u = att_unit(op, r, k);
          for (int pg = u.pg0; pg < u.pg1; ++pg) {
            cur_next(cur, att_stage_bytes(pb), RB);
            const int b = (int)(cur.i % kNB);
            const bool first = pg == u.pg0;
            if (lane == 0) {
              mbar_wait(&ready[b], (uint32_t)((cur.i / kNB) & 1));
              if (first) mbar_expect_tx(&full[b], (uint32_t)op.G * kD * 2);
              else mbar_arrive(&full[b]);
            }
            __syncwarp();
            if (first && lane < op.G)
              bulk_g2s(ring + cur.off + 2 * pb + lane * kQPitch,
                       op.q + (long long)u.b * op.q_stride + (long long)(u.g * op.G + lane) * kD, kD * 2, &full[b]);
          }
        }
      }
    }
  } else {
    // ======================================================== consumers
    const int t = threadIdx.x - 64;
    const int cw = warp - 2;
    Cur cur{-1, 0, 0};
    const uint32_t ring_u = su32(ring);
    for (int oi = 0; oi < P.n_ops; ++oi) {
      if (cw == 0)
        for (int k = lane; k < (int)(sizeof(Op) / 16); k += 32)
          reinterpret_cast<int4*>(sop)[k] = reinterpret_cast<const int4*>(P.ops + oi)[k];
      named_sync(1, kConsumers);
      const Op& op = *sop;
      if (op.type == DAK_STEP_LINEAR) {
        const LinRole r = lin_role(op, cta);
        float st_sum = 0.f, st_sq = 0.f;  // LN statistics of this CTA's outputs (thread n < N)
        if (r.active) {
          const int kc = op.kc, nch = (int)(op.K / kc);
          const int KS = kc >> 4;
          const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
          const int WM = kConsumerWarps / WK;
          const int wk = cw % WK, wm = cw / WK;
          const int nks = KS / WK;
          const uint32_t row_bytes = (uint32_t)kc * 2;
          const uint32_t a_step = (uint32_t)(WM * 16) * row_bytes;
          const int ahalf = lane >> 4;
          const int pitch = kc * 2 + 16;
          const uint32_t b_base = (uint32_t)((lane & 7) + ((lane >> 4) << 3)) * pitch + ((lane >> 3) & 1) * 16;
          for (long long r0 = r.rb; r0 < r.re; r0 += op.rb_rows) {
            const int R = (int)min((long long)op.rb_rows, r.re - r0);
            const int MT = (R + 15) >> 4;
            const int mtw = (MT + WM - 1) / WM;
            const uint32_t a_base = (uint32_t)(wm * 16 + (lane & 15)) * row_bytes;
            const int key = (int)((r0 + wm * 16 + (lane & 15)) & 7);
            float acc[kMtwMax][NT][4];
#pragma unroll
            for (int a = 0; a < kMtwMax; ++a)
#pragma unroll
              for (int b = 0; b < NT; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
            // epilogue operands preloaded right after the first stage lands (its full barrier
            // orders us after the producer's dependency acquire), so their L2 latency hides under
            // the stage loop: thread t owns epilogue elements q = t + i*256 -> (n = q/R, rr = q%R)
            constexpr int kEpi = 8;
            const long long row0 = r.host ? r0 : op.h + r0;
            const int RN = R * N;
            float pre_bias[kEpi], pre_res[kEpi];
            __nv_bfloat16* pre_kv[kEpi];
            auto kv_target = [&](int n, long long m) -> __nv_bfloat16* {
              // rows from kv_row0: kv_kind 3 = [k rows; v rows] (fused QKV), 1 = k rows, 2 = v rows
              const long long kvr = m - op.kv_row0;
              const int hd = op.Hkv * kD;
              const bool isv = op.kv_kind == 2 || (op.kv_kind == 3 && kvr >= hd);
              const int col = (int)(op.kv_kind == 3 && isv ? kvr - hd : kvr);
              const int gk = col / kD, dd = col % kD;
              const int ps = op.positions[n];
              const uint32_t e = (uint32_t)op.block_table[(long long)n * op.max_pages + ps / op.page];
              const long long idx = (long long)(e & ~kHostBit);
              char* pool = (e & kHostBit) ? (isv ? op.v_host : op.k_host) : (isv ? op.v_hbm : op.k_hbm);
              return reinterpret_cast<__nv_bfloat16*>(pool + (idx * op.Hkv + gk) * (long long)op.page * kD * 2 +
                                                      pg_off(ps % op.page, dd >> 3) + (dd & 7) * 2);
            };
            const int sz = lin_stage_bytes(R, kc, N8);
            const uint32_t xo = (uint32_t)lin_stage_w(R, kc);
            for (int c = 0; c < nch; ++c) {
              cur_next(cur, sz, RB);
              const int sb = (int)(cur.i % kNB);
              mbar_wait(&full[sb], (uint32_t)((cur.i / kNB) & 1));
              if (c == 0) {
                if (r0 == r.rb && t == 0) DAK_TRACE(oi, 2);
#pragma unroll
                for (int i = 0; i < kEpi; ++i) {
                  const int q = t + i * kConsumers;
                  pre_bias[i] = 0.f;
                  pre_res[i] = 0.f;
                  pre_kv[i] = nullptr;
                  if (q < RN) {
                    const int n = q / R, rr = q - n * R;
                    const long long m = row0 + rr;
                    if (op.bias) pre_bias[i] = __bfloat162float(op.bias[m]);
                    if (op.residual) pre_res[i] = __bfloat162float(op.residual[(long long)n * op.ldy + m]);
                    if (op.kv_row0 >= 0 && m >= op.kv_row0) pre_kv[i] = kv_target(n, m);
                  }
                }
              }
              const uint32_t ws = ring_u + (uint32_t)cur.off + a_base;
              const uint32_t xs = ring_u + (uint32_t)cur.off + xo + b_base;
              switch (mtw) {
                case 1: mma_stage<NT, 1>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                case 2: mma_stage<NT, 2>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                case 3: mma_stage<NT, 3>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                case 4: mma_stage<NT, 4>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                case 5:
                case 6: mma_stage<NT, 6>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                case 7:
                case 8: mma_stage<NT, 8>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
                default: mma_stage<NT, 12>(acc, ws, xs, kc, wk, WK, nks, a_step, key, ahalf); break;
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&empty[sb]);
            }
            // cross-warp reduction in fixed wk order. Fast form: every warp writes its partial
            // tile into its own slice [wk][R][N], one barrier, then each element sums the slices
            // in order 0..WK-1 (same association as the round-robin form, one barrier not WK).
            const int g = lane >> 2, c2 = (lane & 3) * 2;
            const bool sliced = WK * RN * 4 <= kScratch;
            for (int round = 0; round < (sliced ? 1 : WK); ++round) {
              if (sliced || wk == round) {
#pragma unroll
                for (int mi = 0; mi < kMtwMax; ++mi) {
                  const int mt = wm + WM * mi;
                  if (mi < mtw && mt < MT) {
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                      for (int cc = 0; cc < 4; ++cc) {
                        const int rr = mt * 16 + g + (cc >> 1) * 8;
                        const int n = nt * 8 + c2 + (cc & 1);
                        if (rr < R && n < N) {
                          if (sliced) {
                            scratch[(wk * R + rr) * N + n] = acc[mi][nt][cc];
                          } else {
                            float* q = &scratch[rr * N + n];
                            *q = round == 0 ? acc[mi][nt][cc] : *q + acc[mi][nt][cc];
                          }
                        }
                      }
                  }
                }
              }
              named_sync(1, kConsumers);
            }
            // epilogue: bias, act, residual, bf16 store, fused KV append
            for (int q = t, i = 0; q < RN; q += kConsumers, ++i) {
              const int n = q / R, rr = q - n * R;
              float v = scratch[rr * N + n];
              if (sliced)
                for (int w = 1; w < WK; ++w) v += scratch[(w * R + rr) * N + n];
              const long long m = row0 + rr;
              float bsv = 0.f, rsv = 0.f;
              __nv_bfloat16* kvp = nullptr;
              if (i < kEpi) {
#pragma unroll
                for (int j = 0; j < kEpi; ++j)
                  if (j == i) {
                    bsv = pre_bias[j];
                    rsv = pre_res[j];
                    kvp = pre_kv[j];
                  }
              } else {
                if (op.bias) bsv = __bfloat162float(op.bias[m]);
                if (op.residual) rsv = __bfloat162float(op.residual[(long long)n * op.ldy + m]);
                if (op.kv_row0 >= 0 && m >= op.kv_row0) kvp = kv_target(n, m);
              }
              v += bsv;
              if (op.act == DAK_ACT_RELU) v = fmaxf(v, 0.f);
              v += rsv;
              const __nv_bfloat16 o = __float2bfloat16_rn(v);
              op.y[(long long)n * op.ldy + m] = o;
              scratch[rr * N + n] = __bfloat162float(o);  // stored value (for LN statistics)
              if (kvp) *kvp = o;
            }
            named_sync(1, kConsumers);
            if (op.stats_out && t < N) {
              for (int rr = 0; rr < R; ++rr) {
                const float v = scratch[rr * N + t];
                st_sum += v;
                st_sq += v * v;
              }
            }
            named_sync(1, kConsumers);
          }
        }
        if (op.stats_out && t < N) {
          op.stats_out[((long long)cta * N + t) * 2] = st_sum;
          op.stats_out[((long long)cta * N + t) * 2 + 1] = st_sq;
        }
      } else if (op.type == DAK_STEP_ATTENTION) {
        const AttRole r = att_role(op, cta);
        const int gq = lane >> 2, cq = lane & 3;
        const int pb = op.page * kD * 2;
        const int tiles_per_page = op.page / 16;
        for (int k = r.j; k < r.n_units; k += r.n) {
          const Unit u = att_unit(op, r, k);
          const int tok_base = u.pg0 * op.page;
          uint32_t qb[kD / 16][2];
          float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
          float o[kD / 16][4];
#pragma unroll
          for (int i = 0; i < kD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
          for (int pg = u.pg0; pg < u.pg1; ++pg) {
            cur_next(cur, att_stage_bytes(pb), RB);
            const int sb = (int)(cur.i % kNB);
            mbar_wait(&full[sb], (uint32_t)((cur.i / kNB) & 1));
            if (k == r.j && pg == u.pg0 && t == 0) DAK_TRACE(oi, 2);
            if (pg == u.pg0) {
              const uint32_t qs = ring_u + (uint32_t)cur.off + 2 * pb;
#pragma unroll
              for (int ks = 0; ks < kD / 16; ++ks)
                ldsm_x2(qs + (lane & 7) * kQPitch + (2 * ks + ((lane >> 3) & 1)) * 16, qb[ks][0], qb[ks][1]);
            }
            const uint32_t kbase = ring_u + (uint32_t)cur.off;
            const uint32_t vbase = kbase + pb;
            for (int tl = 0; tl < tiles_per_page; ++tl) {
              const int tile = (pg - u.pg0) * tiles_per_page + tl;
              if ((tile & (kConsumerWarps - 1)) != cw) continue;
              const int tok0 = tok_base + tile * 16;
              if (tok0 >= u.L) continue;
              const int r0 = tl * 16;
              float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int ks = 0; ks < kD / 16; ++ks) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4(kbase + pg_off(r0 + (lane & 15), 2 * ks + (lane >> 4)), a0, a1, a2, a3);
                mma_bf16(sc, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
              }
              const bool v0 = tok0 + gq < u.L, v1 = tok0 + gq + 8 < u.L;
              const float s0 = v0 ? sc[0] * op.scale_log2 : -INFINITY;
              const float s1 = v0 ? sc[1] * op.scale_log2 : -INFINITY;
              const float s2 = v1 ? sc[2] * op.scale_log2 : -INFINITY;
              const float s3 = v1 ? sc[3] * op.scale_log2 : -INFINITY;
              float mx0 = fmaxf(s0, s2), mx1 = fmaxf(s1, s3);
#pragma unroll
              for (int off = 4; off < 32; off <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
              }
              const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
              const float al0 = exp2f(m[0] - mn0), al1 = exp2f(m[1] - mn1);
              m[0] = mn0;
              m[1] = mn1;
              const float p0 = exp2f(s0 - mn0), p1 = exp2f(s1 - mn1), p2 = exp2f(s2 - mn0), p3 = exp2f(s3 - mn1);
              l[0] = l[0] * al0 + (p0 + p2);
              l[1] = l[1] * al1 + (p1 + p3);
#pragma unroll
              for (int i = 0; i < kD / 16; ++i) {
                o[i][0] *= al0; o[i][1] *= al1; o[i][2] *= al0; o[i][3] *= al1;
              }
              const uint32_t b0 = movm_t(pack_bf16(p0, p1));
              const uint32_t b1 = movm_t(pack_bf16(p2, p3));
#pragma unroll
              for (int i = 0; i < kD / 16; ++i) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vbase + pg_off(r0 + (lane & 7) + ((lane >> 4) << 3), 2 * i + ((lane >> 3) & 1)), a0, a1, a2, a3);
                mma_bf16(o[i], a0, a1, a2, a3, b0, b1);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[sb]);
          }
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            l[0] += __shfl_xor_sync(0xffffffffu, l[0], off);
            l[1] += __shfl_xor_sync(0xffffffffu, l[1], off);
          }
          float* so = scratch + cw * (kGmax * kD + 2 * kGmax);
          float* sm = so + kGmax * kD;
#pragma unroll
          for (int i = 0; i < kD / 16; ++i) {
            const int d0 = 16 * i + gq;
            so[(2 * cq) * kD + d0] = o[i][0];
            so[(2 * cq + 1) * kD + d0] = o[i][1];
            so[(2 * cq) * kD + d0 + 8] = o[i][2];
            so[(2 * cq + 1) * kD + d0 + 8] = o[i][3];
          }
          if (gq == 0) {
            sm[2 * cq] = m[0];
            sm[2 * cq + 1] = m[1];
            sm[kGmax + 2 * cq] = l[0];
            sm[kGmax + 2 * cq + 1] = l[1];
          }
          named_sync(1, kConsumers);
          const int npg = (u.L + op.page - 1) / op.page;
          const int nch = (npg + op.chunk_pages - 1) / op.chunk_pages;
          const long long ubase = (((long long)u.b * op.Hkv + u.g) * op.max_chunks + u.c) * op.G;
          for (int i = t; i < op.G * kD; i += kConsumers) {
            const int hh = i / kD, d = i % kD;
            float M = -INFINITY;
            for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, scratch[w * (kGmax * kD + 2 * kGmax) + kGmax * kD + hh]);
            float Ls = 0.f, Os = 0.f;
            for (int w = 0; w < kConsumerWarps; ++w) {
              const float* ww = scratch + w * (kGmax * kD + 2 * kGmax);
              const float mw = ww[kGmax * kD + hh];
              if (mw == -INFINITY) continue;
              const float sc = exp2f(mw - M);
              Ls += ww[kGmax * kD + kGmax + hh] * sc;
              Os += ww[hh * kD + d] * sc;
            }
            if (nch == 1) {  // single-chunk request: final output straight away
              op.out[((long long)u.b * op.Hq + u.g * op.G + hh) * kD + d] = __float2bfloat16_rn(Os / Ls);
            } else {
              op.part_o[(ubase + hh) * kD + d] = Os / Ls;
              if (d == 0) op.part_lse[ubase + hh] = M + log2f(Ls);
            }
          }
          named_sync(1, kConsumers);
        }
      } else if (op.type == DAK_STEP_COMBINE) {
        if (t == 0) spin_until_geq(&P.done[op.dep], G);
        named_sync(1, kConsumers);
        __threadfence();
        const int total = op.cols * op.Hq;  // cols = B
        for (int bh = cta; bh < total; bh += G) {
          const int b = bh / op.Hq, h = bh % op.Hq;
          const int L = op.seq_lens[b];
          const int npg = (L + op.page - 1) / op.page;
          const int nch = (npg + op.chunk_pages - 1) / op.chunk_pages;
          if (nch == 1) continue;
          const int g = h / op.G, hh = h % op.G;
          const long long base = (((long long)b * op.Hkv + g) * op.max_chunks) * op.G + hh;
          float M = -INFINITY;
          for (int c = 0; c < nch; ++c) M = fmaxf(M, op.part_lse[base + (long long)c * op.G]);
          for (int d = t; d < kD; d += kConsumers) {
            float num = 0.f, den = 0.f;
            for (int c = 0; c < nch; ++c) {
              const float w = exp2f(op.part_lse[base + (long long)c * op.G] - M);
              den += w;
              num += w * op.part_o[(base + (long long)c * op.G) * kD + d];
            }
            op.out[((long long)b * op.Hq + h) * kD + d] = __float2bfloat16_rn(num / den);
          }
        }
      } else if (op.type == DAK_STEP_LAYERNORM || op.type == DAK_STEP_EMBED) {
        if (op.type == DAK_STEP_LAYERNORM) {
          if (t == 0 && op.dep >= 0) spin_until_geq(&P.done[op.dep], G);
          if (t == 0) DAK_TRACE(oi, 1);
          named_sync(1, kConsumers);
          __threadfence();
          // fixed-order parallel reduction of the per-CTA partial statistics: warp w owns rows
          // w, w+8; lane l sums partials l, l+32, ... then a fixed xor tree (deterministic)
          for (int n = cw; n < N; n += kConsumerWarps) {
            double sm = 0.0, sq = 0.0;
            for (int c = lane; c < G; c += 32) {
              sm += op.stats_in[((long long)c * N + n) * 2];
              sq += op.stats_in[((long long)c * N + n) * 2 + 1];
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              sm += __shfl_xor_sync(0xffffffffu, sm, off);
              sq += __shfl_xor_sync(0xffffffffu, sq, off);
            }
            if (lane == 0) {
              const double mean = sm / op.cols;
              double var = sq / op.cols - mean * mean;
              if (var < 0.0) var = 0.0;
              s_stat[2 * n] = (float)mean;
              s_stat[2 * n + 1] = (float)(1.0 / sqrt(var + (double)op.eps));
            }
          }
          named_sync(1, kConsumers);
        }
        const int c0 = (int)((long long)cta * op.cols / G), c1 = (int)((long long)(cta + 1) * op.cols / G);
        const int w = c1 - c0;
        float psum = 0.f, psq = 0.f;
        for (int i = t; i < N * w; i += kConsumers) {
          const int n = i / w, c = c0 + i % w;
          float v;
          if (op.type == DAK_STEP_LAYERNORM) {
            v = (__bfloat162float(op.x[(long long)n * op.cols + c]) - s_stat[2 * n]) * s_stat[2 * n + 1];
            v = v * __bfloat162float(op.ln_w[c]) + (op.ln_b ? __bfloat162float(op.ln_b[c]) : 0.f);
          } else {
            const long long tk = op.tokens[n];
            v = __bfloat162float(op.tok_emb[tk * op.cols + c]);
            if (op.pos_emb) v += __bfloat162float(op.pos_emb[((long long)op.positions[n] + op.pos_offset) * op.cols + c]);
          }
          const __nv_bfloat16 o = __float2bfloat16_rn(v);
          op.y[(long long)n * op.cols + c] = o;
          if (op.stats_out) scratch[i] = __bfloat162float(o);
        }
        if (op.stats_out) {
          named_sync(1, kConsumers);
          if (t < N) {
            for (int c = 0; c < w; ++c) {
              const float v = scratch[t * w + c];
              psum += v;
              psq += v * v;
            }
            op.stats_out[((long long)cta * N + t) * 2] = psum;
            op.stats_out[((long long)cta * N + t) * 2 + 1] = psq;
          }
        }
      }
      // ---- op complete for this CTA: publish (gpu-scope release)
      named_sync(1, kConsumers);
      if (t == 0) {
        __threadfence();
        DAK_TRACE(oi, 3);
        red_release_add(&P.done[oi], 1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(P.finished, 1);
    if (prev == G - 1) {  // last CTA out: reset the counters for the next launch
      for (int i = 0; i < P.n_ops; ++i) P.done[i] = 0;
      __threadfence();
      *P.finished = 0;
    }
  }
}

// ---------------------------------------------------------------------------------- host side
static inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
static const int kMtwBuckets[] = {1, 2, 3, 4, 6, 8, 12};
static int mtw_bucket(int need) {
  for (int b : kMtwBuckets)
    if (b >= need) return b;
  return -1;
}

// largest row block R <= rmax within the MMA accumulator capacity whose weight bytes per stage
// stay <= kStageW (stages beyond that only cost ring depth)
constexpr int kStageW = 48 * 1024;
static int row_block(int kc, long long rmax) {
  const int KS = kc / 16;
  const int WK = KS < kConsumerWarps ? KS : kConsumerWarps;
  const int WM = kConsumerWarps / WK;
  int best = 0;
  for (int R = 16; R <= 16 * WM * kMtwMax; R += 16) {
    const int need = (int)cdiv(cdiv(R, 16), WM);
    const int b = mtw_bucket(need);
    if (b < 0) break;
    if ((long long)R * kc * 2 <= kStageW) best = R;
  }
  if (best == 0) return 0;
  return (int)std::min<long long>(best, std::max<long long>(16, rmax));
}

}  // namespace step
}  // namespace dak

using namespace dak;

extern "C" {

int32_t dak_step_choose_kc(int64_t rows_per_cta, int64_t K) {
  // the widest KC whose row block holds all of a CTA's rows in one slot (fewest, largest stages)
  for (int kc = 256; kc >= 64; kc >>= 1)
    if (K % kc == 0 && step::row_block(kc, rows_per_cta) >= rows_per_cta) return kc;
  return 64;
}

size_t dak_step_buffer_bytes(int32_t n_ops) {
  return (size_t)n_ops * sizeof(step::Op) + (size_t)(n_ops + 32) * sizeof(int);
}

dak_status dak_step_compile(const dak_step_op* ops, int32_t n_ops, int32_t N, const dak_launch_cfg* cfg, void* dev_buf,
                            size_t dev_bytes, dak_step_plan* out) {
  if (!ops || n_ops <= 0 || !dev_buf || !out || N <= 0) return fail(DAK_EINVAL, "dak_step_compile: bad arguments");
  if (N > 16) return fail(DAK_EUNSUPPORTED, "dak_step_compile: N > 16");
  if (dev_bytes < dak_step_buffer_bytes(n_ops)) return fail(DAK_EINVAL, "dak_step_compile: device buffer too small");
  int sms = 0;
  dak_status st = dak_device_sms(&sms);
  if (st != DAK_OK) return st;
  const dak_launch_cfg c = cfg ? *cfg : dak_launch_cfg{};
  const int G = sms;
  std::vector<step::Op> dv(n_ops);
  static_assert(sizeof(step::Op) <= 512, "op descriptor copy slot");
  const int ring_bytes = step::kSmemBudget - step::kHeader - step::kScratch - step::kL1Reserve;
  long long max_stage = 0;
  for (int i = 0; i < n_ops; ++i) {
    const dak_step_op& s = ops[i];
    step::Op& o = dv[i];
    o = step::Op{};
    o.type = s.type;
    o.dep = s.dep;
    if (s.dep >= i) return fail(DAK_EINVAL, "dak_step_compile: op %d depends on a later op", i);
    o.act = s.act;
    o.x = (const __nv_bfloat16*)s.x;
    o.y = (__nv_bfloat16*)s.y;
    o.ldy = s.ldy > 0 ? s.ldy : s.M;
    o.bias = (const __nv_bfloat16*)s.bias;
    o.residual = (const __nv_bfloat16*)s.residual;
    o.stats_out = s.stats_out;
    o.kv_row0 = s.kv_kind > 0 ? s.kv_row0 : -1;
    o.kv_kind = s.kv_kind;
    if (s.kv_kind < 0 || s.kv_kind > 3) return fail(DAK_EINVAL, "op %d: bad kv_kind", i);
    o.stats_in = s.stats_in;
    o.ln_w = (const __nv_bfloat16*)s.ln_w;
    o.ln_b = (const __nv_bfloat16*)s.ln_b;
    o.eps = s.eps;
    o.cols = s.cols;
    o.tokens = s.tokens;
    o.positions = s.positions;
    o.tok_emb = (const __nv_bfloat16*)s.tok_emb;
    o.pos_emb = (const __nv_bfloat16*)s.pos_emb;
    o.pos_offset = s.pos_offset;
    o.q = (const __nv_bfloat16*)s.q;
    o.out = (__nv_bfloat16*)s.out;
    o.k_hbm = (char*)s.k_hbm;
    o.v_hbm = (char*)s.v_hbm;
    o.k_host = (char*)s.k_host;
    o.v_host = (char*)s.v_host;
    o.block_table = s.block_table;
    o.seq_lens = s.seq_lens;
    o.Hq = s.Hq;
    o.Hkv = s.Hkv;
    o.page = s.page_size;
    o.max_pages = s.max_pages;
    o.chunk_pages = s.chunk_pages;
    o.part_o = s.part_o;
    o.part_lse = s.part_lse;
    o.units_host = s.units_host;
    o.units_hbm = s.units_hbm;
    o.n_units_host = s.n_units_host;
    o.n_units_hbm = s.n_units_hbm;
    if (s.type == DAK_STEP_LINEAR) {
      if (s.M <= 0 || s.K <= 0 || s.h < 0 || s.h > s.M || s.K % 64) return fail(DAK_EINVAL, "op %d: bad linear shape", i);
      if (s.kc < 64 || (s.kc & (s.kc - 1)) || s.K % s.kc || s.kc > 256)
        return fail(DAK_EINVAL, "op %d: kc must be a power of two in [64,256] dividing K", i);
      if (!s.x || !s.y || (s.h > 0 && !s.w_host) || (s.h < s.M && !s.w_hbm)) return fail(DAK_EINVAL, "op %d: NULL", i);
      o.w_host = (const char*)s.w_host;
      o.w_hbm = (const char*)s.w_hbm;
      o.M = s.M; o.K = s.K; o.h = s.h; o.kc = s.kc;
      o.n_host = s.h > 0 ? std::max(1, s.n_cta_host > 0 ? s.n_cta_host : c.n_cta_host > 0 ? c.n_cta_host : 1) : 0;
      o.n_hbm = G - o.n_host;
      if (o.n_hbm <= 0 && s.h < s.M) return fail(DAK_EINVAL, "op %d: no HBM CTAs left", i);
      const long long rmax = std::max(o.n_host ? step::cdiv(s.h, o.n_host) : 0, o.n_hbm ? step::cdiv(s.M - s.h, o.n_hbm) : 0);
      const int rb_max = step::row_block(s.kc, rmax);
      if (rb_max <= 0) return fail(DAK_EUNSUPPORTED, "op %d: no row block fits kc=%d", i, s.kc);
      // equal-size row blocks (no small trailing block with tiny stages)
      const long long nblk = step::cdiv(std::max<long long>(rmax, 1), rb_max);
      o.rb_rows = (int)std::min<long long>(rb_max, step::cdiv(step::cdiv(std::max<long long>(rmax, 1), nblk), 16) * 16);
      const long long stage = step::cdiv((long long)o.rb_rows * s.kc * 2, 128) * 128 +
                              step::cdiv(step::cdiv(N, 8) * 8 * (s.kc * 2 + 16), 128) * 128;
      max_stage = std::max(max_stage, stage);
      int win = step::kNB;
      if (c.window > 0) win = c.window;
      else if (c.congestion_control) {
        const long long hst = std::max<long long>(1, std::min<long long>(o.rb_rows, step::cdiv(s.h, std::max(1, o.n_host))) * s.kc * 2);
        win = (int)std::max<long long>(1, step::cdiv(192 * 1024, hst * std::max(1, o.n_host)));
      }
      o.window = win;
      if (s.kv_row0 >= 0 && (!s.positions || !s.block_table || s.Hkv <= 0 || s.page_size <= 0))
        return fail(DAK_EINVAL, "op %d: fused KV append needs positions, block table, pools", i);
    } else if (s.type == DAK_STEP_ATTENTION || s.type == DAK_STEP_COMBINE) {
      if (s.Hq <= 0 || s.Hkv <= 0 || s.Hq % s.Hkv || s.Hq / s.Hkv > step::kGmax || s.d != step::kD ||
          s.page_size % 16 || s.page_size > 256 || s.chunk_pages <= 0)
        return fail(DAK_EUNSUPPORTED, "op %d: attention shape outside this build (d=128, Hq/Hkv<=8, page<=256)", i);
      max_stage = std::max<long long>(max_stage, 2LL * s.page_size * step::kD * 2 + step::kGmax * step::kQPitch);
      o.G = s.Hq / s.Hkv;
      o.max_chunks = (int)step::cdiv(s.max_pages, s.chunk_pages);
      o.q_stride = s.q_stride > 0 ? s.q_stride : (long long)s.Hq * step::kD;
      const float scale = s.scale > 0.f ? s.scale : 1.0f / sqrtf((float)step::kD);
      o.scale_log2 = scale * 1.4426950408889634f;
      o.n_host = s.n_units_host > 0 ? std::max(1, s.n_cta_host > 0 ? s.n_cta_host : c.n_cta_host > 0 ? c.n_cta_host : 1) : 0;
      o.n_hbm = G - o.n_host;
      o.window = step::kNB;
      if (c.window > 0) o.window = c.window;
      else if (c.congestion_control)
        o.window = (int)std::max<long long>(1, step::cdiv(192 * 1024, (long long)s.page_size * step::kD * 4 * std::max(1, o.n_host)));
      if (s.type == DAK_STEP_COMBINE) o.cols = s.cols;  // = B
      if (s.dep < 0 && s.type == DAK_STEP_ATTENTION) return fail(DAK_EINVAL, "op %d: attention needs a dependency", i);
    } else if (s.type == DAK_STEP_LAYERNORM || s.type == DAK_STEP_EMBED) {
      if (s.cols <= 0 || !s.y || (s.type == DAK_STEP_LAYERNORM && (!s.x || !s.stats_in || !s.ln_w)) ||
          (s.type == DAK_STEP_EMBED && (!s.tokens || !s.tok_emb)))
        return fail(DAK_EINVAL, "op %d: bad layernorm/embed", i);
      if ((long long)N * step::cdiv(s.cols, G) * 4 > step::kScratch)
        return fail(DAK_EUNSUPPORTED, "op %d: columns per CTA too many", i);
    } else {
      return fail(DAK_EINVAL, "op %d: unknown type %d", i, s.type);
    }
  }
  if (2 * max_stage > ring_bytes) return fail(DAK_EUNSUPPORTED, "dak_step_compile: a %lld B stage does not fit twice", max_stage);
  for (auto& o : dv)
    if (o.window > step::kNB) o.window = step::kNB;
  out->dev = dev_buf;
  out->n_ops = n_ops;
  out->N = N;
  out->grid = G;
  out->ring_bytes = ring_bytes;
  out->off_scratch = step::kHeader + ring_bytes;
  out->smem = out->off_scratch + step::kScratch;
  out->pdl = c.pdl;
  DAK_CUDA_TRY(cudaMemcpy(dev_buf, dv.data(), sizeof(step::Op) * n_ops, cudaMemcpyHostToDevice));
  DAK_CUDA_TRY(cudaMemset((char*)dev_buf + sizeof(step::Op) * n_ops, 0, (size_t)(n_ops + 32) * sizeof(int)));
  return DAK_OK;
}

dak_status dak_step_launch(const dak_step_plan* pl, dak_stream_t stream) {
  if (!pl || !pl->dev) return fail(DAK_EINVAL, "dak_step_launch: NULL plan");
  step::Params P;
  P.ops = (const step::Op*)pl->dev;
  P.n_ops = pl->n_ops;
  P.N = pl->N;
  P.ring_bytes = pl->ring_bytes;
  P.done = (int*)((char*)pl->dev + sizeof(step::Op) * pl->n_ops);
  P.finished = P.done + pl->n_ops;
  P.off_scratch = pl->off_scratch;
  P.trace = (unsigned long long*)pl->trace;
  const void* fn = pl->N <= 8 ? (const void*)step::step_kernel<1> : (const void*)step::step_kernel<2>;
  static int attr_set[2] = {0, 0};
  int& set = attr_set[pl->N <= 8 ? 0 : 1];
  if (!set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, step::kSmemBudget));
    set = 1;
  }
  void* args[] = {&P};
  // cooperative launch: all CTAs co-resident (the completion-counter waits require it)
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl->grid);
  cfg.blockDim = dim3(step::kThreads);
  cfg.dynamicSmemBytes = pl->smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  return DAK_OK;
}

}  // extern "C"
