// dak_attention — split paged GQA decode attention for sm_100a (PAPER §4, §3.1).
//
// The KV cache is paged; each page of one kv head is a [page_size, d] bf16 block living either in
// the HBM pool or in the pinned, device-mapped host pool (block-table bit 31 selects the tier).
// Work is split flash-decoding style into units (request b, kv head g, chunk c of chunk_pages
// pages). Each CTA reads exactly one tier: CTAs [0, n_host) take the units whose chunk
// starts on a host page, the rest take HBM units, round-robin by the unit's rank within its tier.
// A producer lane streams the unit's K and V pages into an SMEM ring with 1-D bulk copies
// (cp.async.bulk, the TMA engine) completing on mbarriers, host stages capped by the congestion
// window. Eight consumer warps compute on tensor cores (mma.sync m16n8k16 bf16->fp32):
//   S^T[16 tokens x 8 heads] = K_tile . Q^T       (all q heads of the GQA group in one n8 tile)
//   online softmax per head (exp2 domain), P^T fed back as the B operand via movmatrix.trans
//   O^T[d x 8 heads]       += V_tile^T . P^T      (ldmatrix.trans on the swizzled V page)
// Warps own 16-token tiles (tile t -> warp t mod 8); at the end of a unit their (m, l, O) are
// merged in fixed warp order and the normalised partial (o, log2-sum-exp) goes to workspace.
// A combine kernel merges the chunk partials of each (b, q-head) in chunk order -> bf16 output.
// Every reduction order is fixed by (seq_len, chunk_pages, page_size): outputs are independent
// of which pages live on the host (bitwise r-invariance).
//
// KV page layout ("DAK-PG"): a page of one kv head is [page_size][d] bf16 with the 16-byte chunk
// j of token row t stored at chunk ((j>>3)<<3) | ((j&7) ^ (t&7)) (bank-conflict-free ldmatrix).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace dak {
namespace attn {

constexpr int kD = 128;
constexpr int kGmax = 8;              // q heads per kv head handled in one n8 tile
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = 32 + kConsumers;
constexpr int kMaxStages = 8;
constexpr int kQPitch = kD * 2 + 16;  // bytes per q row in smem
constexpr int kMaxPairs = 8192;       // (request, chunk) pairs scheduled per launch
constexpr int kSmemBudget = 226 * 1024;  // 227 KB opt-in minus the kernel's static scan scratch
constexpr uint32_t kHostBit = 0x80000000u;

struct Params {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  const char* k_hbm;
  const char* v_hbm;
  const char* k_host;
  const char* v_host;
  const int* block_table;
  const int* seq_lens;
  int B, Hq, Hkv, G, page, max_pages, chunk_pages, max_chunks;
  long long q_stride;  // elements between consecutive requests of q
  float scale_log2;  // softmax scale * log2(e)
  float* part_o;     // [B][Hkv][max_chunks][G][d]
  float* part_lse;   // [B][Hkv][max_chunks][G]   (log2 domain)
  int n_host, n_hbm, stages, window;
  int stage_bytes;   // K page + V page
  int off_q, off_scratch, off_pairs;
  unsigned long long* trace;   // dak_trace_enable slots (nullable): split kernel, combine kernel
  unsigned long long* trace2;
};

__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 4 + k] = t;
  }
}

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
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of 16-byte chunk j of token row t in a DAK-PG page (row pitch 256 B)
__device__ __forceinline__ uint32_t pg_off(int t, int j) {
  return (uint32_t)(t * (kD * 2) + ((((j >> 3) << 3) | ((j & 7) ^ (t & 7))) << 4));
}

// Unit k of a tier -> (pair index, kv head). pref[p] = tier-matching pairs before pair p.
__device__ __forceinline__ int find_pair(const int* pref, int n_pairs, int rank) {
  int lo = 0, hi = n_pairs - 1;  // largest p with pref[p] <= rank and pair p matching
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= rank) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads, 1) split_attention_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  int* s_count = reinterpret_cast<int*>(empty + kMaxStages);
  unsigned char* ring = smem + 1024;
  unsigned char* qring = smem + p.off_q;  // [stages][kGmax][kD] bf16: q of the unit starting in that stage
  float* scratch = reinterpret_cast<float*>(smem + p.off_scratch);
  int* pref = reinterpret_cast<int*>(smem + p.off_pairs);

  const int cta = blockIdx.x;
  const bool host = cta < p.n_host;
  const int my_j = host ? cta : cta - p.n_host;
  const int my_n = host ? p.n_host : p.n_hbm;
  const int slots = host ? p.window : p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int page_bytes = p.page * kD * 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tstamp(p.trace, 0);
  }
  // q rows >= G of every slot stay zero (the bulk copies write rows < G only)
  for (int i = threadIdx.x; i < p.stages * kGmax * kD / 8; i += kThreads)
    reinterpret_cast<uint4*>(qring)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  grid_dep_launch();
  grid_dep_wait();  // block table, seq_lens and q come from earlier kernels
  if (threadIdx.x == 0) tstamp(p.trace, 1);
  // ---- schedule: pairs (b, c) linearised p = b*max_chunks + c; tier = bit 31 of the chunk's first page
  const int n_pairs = p.B * p.max_chunks;
  // flags -> exclusive prefix over tier-matching pairs (block-wide, fixed order)
  {
    __shared__ int warp_tot[kThreads / 32];
    int carry = 0;
    for (int base = 0; base < n_pairs; base += kThreads) {
      const int i = base + threadIdx.x;
      int f = 0;
      if (i < n_pairs) {
        const int b = i / p.max_chunks, c = i % p.max_chunks;
        const int L = p.seq_lens[b];
        const int npg = (L + p.page - 1) / p.page;
        if (c * p.chunk_pages < npg) {
          const uint32_t e = (uint32_t)p.block_table[(long long)b * p.max_pages + c * p.chunk_pages];
          f = ((e & kHostBit) != 0) == host;
        }
      }
      // inclusive warp scan
      int v = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) warp_tot[warp] = v;
      __syncthreads();
      int before = carry;
      for (int w = 0; w < warp; ++w) before += warp_tot[w];
      if (i < n_pairs) pref[i] = before + v - f;  // exclusive
      int tot = 0;
      for (int w = 0; w < kThreads / 32; ++w) tot += warp_tot[w];
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) *s_count = carry;
    __syncthreads();
  }
  const int n_units = *s_count * p.Hkv;

  if (warp == 0) {
    // ================================ producer
    if (lane == 0) {
      int it = 0;
      for (int k = my_j; k < n_units; k += my_n) {
        const int pr = find_pair(pref, n_pairs, k / p.Hkv);
        const int g = k % p.Hkv;
        const int b = pr / p.max_chunks, c = pr % p.max_chunks;
        const int L = p.seq_lens[b];
        const int npg = (L + p.page - 1) / p.page;
        const int pg0 = c * p.chunk_pages, pg1 = min(npg, pg0 + p.chunk_pages);
        for (int pg = pg0; pg < pg1; ++pg, ++it) {
          const int s = it % slots;
          if (it >= slots) mbar_wait(&empty[s], ((uint32_t)(it / slots) & 1u) ^ 1u);
          const uint32_t e = (uint32_t)p.block_table[(long long)b * p.max_pages + pg];
          const long long idx = (long long)(e & ~kHostBit);
          const bool eh = (e & kHostBit) != 0;
          const long long off = (idx * p.Hkv + g) * (long long)page_bytes;
          const uint32_t q_bytes = pg == pg0 ? (uint32_t)p.G * kD * 2 : 0u;  // q rides with the first page
          mbar_expect_tx(&full[s], 2u * page_bytes + q_bytes);
          unsigned char* dst = ring + (size_t)s * p.stage_bytes;
          bulk_g2s(dst, (eh ? p.k_host : p.k_hbm) + off, page_bytes, &full[s]);
          bulk_g2s(dst + page_bytes, (eh ? p.v_host : p.v_hbm) + off, page_bytes, &full[s]);
          if (q_bytes)
            bulk_g2s(qring + (size_t)s * kGmax * kD * 2, p.q + (long long)b * p.q_stride + (long long)g * p.G * kD, q_bytes,
                     &full[s]);
        }
      }
    }
    return;
  }

  // ================================ consumers
  const int cw = warp - 1;
  const int t = threadIdx.x - 32;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column pair
  const int tiles_per_page = p.page / 16;
  int it = 0;
  for (int k = my_j; k < n_units; k += my_n) {
    const int pr = find_pair(pref, n_pairs, k / p.Hkv);
    const int g = k % p.Hkv;
    const int b = pr / p.max_chunks, c = pr % p.max_chunks;
    const int L = p.seq_lens[b];
    const int npg = (L + p.page - 1) / p.page;
    const int pg0 = c * p.chunk_pages, pg1 = min(npg, pg0 + p.chunk_pages);
    const int tok_base = pg0 * p.page;  // first token of the chunk
    uint32_t qb[kD / 16][2];

    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    float o[kD / 16][4];
#pragma unroll
    for (int i = 0; i < kD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

    for (int pg = pg0; pg < pg1; ++pg, ++it) {
      const int s = it % slots;
      mbar_wait(&full[s], (uint32_t)(it / slots) & 1u);
      if (pg == pg0) {  // q of the GQA group (prefetched with the unit's first page) -> B fragments
        const uint32_t qsu = su32(qring + (size_t)s * kGmax * kD * 2);
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks)
          ldsm_x2(qsu + (lane & 7) * (kD * 2) + (2 * ks + ((lane >> 3) & 1)) * 16, qb[ks][0], qb[ks][1]);
      }
      const uint32_t kbase = su32(ring + (size_t)s * p.stage_bytes);
      const uint32_t vbase = kbase + page_bytes;
      for (int tl = 0; tl < tiles_per_page; ++tl) {
        const int tile = (pg - pg0) * tiles_per_page + tl;
        if ((tile & (kConsumerWarps - 1)) != cw) continue;
        const int tok0 = tok_base + tile * 16;  // chunk-relative -> absolute token index
        if (tok0 >= L) continue;
        const int r0 = tl * 16;                 // row inside the page
        // ---- S^T = K . Q^T   [16 tokens x 8 heads]
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4(kbase + pg_off(r0 + (lane & 15), 2 * ks + (lane >> 4)), a0, a1, a2, a3);
          mma_bf16(sc, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
        }
        // ---- scale, mask, online softmax (exp2 domain), per head column
        const bool v0 = tok0 + gq < L, v1 = tok0 + gq + 8 < L;
        float s0 = v0 ? sc[0] * p.scale_log2 : -INFINITY;
        float s1 = v0 ? sc[1] * p.scale_log2 : -INFINITY;
        float s2 = v1 ? sc[2] * p.scale_log2 : -INFINITY;
        float s3 = v1 ? sc[3] * p.scale_log2 : -INFINITY;
        float mx0 = fmaxf(s0, s2), mx1 = fmaxf(s1, s3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);  // finite: tile has a valid token
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
        // ---- P^T as B operand: transpose the two 8x8 blocks of P (tokens x heads)
        const uint32_t b0 = movm_t(pack_bf16(p0, p1));
        const uint32_t b1 = movm_t(pack_bf16(p2, p3));
        // ---- O^T[d x heads] += V^T . P^T
#pragma unroll
        for (int i = 0; i < kD / 16; ++i) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(vbase + pg_off(r0 + (lane & 7) + ((lane >> 4) << 3), 2 * i + ((lane >> 3) & 1)), a0, a1, a2, a3);
          mma_bf16(o[i], a0, a1, a2, a3, b0, b1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // ---- warp partials -> scratch [warp][head][d] (+ m, l), then fixed-order merge
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
    consumer_sync();
    const long long ubase = (((long long)b * p.Hkv + g) * p.max_chunks + c) * p.G;
    const bool direct = npg <= p.chunk_pages;  // the request is one chunk: no combine needed
    for (int i = t; i < p.G * kD; i += kConsumers) {
      const int hh = i / kD, d = i % kD;
      float M = -INFINITY;
      for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, scratch[w * (kGmax * kD + 2 * kGmax) + kGmax * kD + hh]);
      float Ls = 0.f, Os = 0.f;
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float* ww = scratch + w * (kGmax * kD + 2 * kGmax);
        const float mw = ww[kGmax * kD + hh];
        if (mw == -INFINITY) continue;  // warp saw no valid token
        const float sc = exp2f(mw - M);
        Ls += ww[kGmax * kD + kGmax + hh] * sc;
        Os += ww[hh * kD + d] * sc;
      }
      if (direct) {
        p.out[((long long)b * p.Hq + g * p.G + hh) * kD + d] = __float2bfloat16_rn(Os / Ls);
      } else {
        p.part_o[(ubase + hh) * kD + d] = Os / Ls;
        if (d == 0) p.part_lse[ubase + hh] = M + log2f(Ls);
      }
    }
    consumer_sync();
    if (t == 0 && k == my_j) tstamp(p.trace, 2);  // first unit done
  }
  if (t == 0) tstamp(p.trace, 3);
}

// merge chunk partials: out[b, h, :] = sum_c w_c o_c, w_c = 2^(lse_c - LSE)   (fixed chunk order)
__global__ void combine_kernel(const Params p) {
  if (threadIdx.x == 0) tstamp(p.trace2, 0);
  grid_dep_launch();
  grid_dep_wait();
  if (threadIdx.x == 0) tstamp(p.trace2, 1);
  const int bh = blockIdx.x;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int g = h / p.G, hh = h % p.G;
  const int L = p.seq_lens[b];
  const int npg = (L + p.page - 1) / p.page;
  const int nch = (npg + p.chunk_pages - 1) / p.chunk_pages;
  if (nch <= 1) {  // written directly by the split kernel
    if (threadIdx.x == 0) tstamp(p.trace2, 3);
    return;
  }
  const long long base = (((long long)b * p.Hkv + g) * p.max_chunks) * p.G + hh;  // + c*G
  float M = -INFINITY;
  for (int c = 0; c < nch; ++c) M = fmaxf(M, p.part_lse[base + (long long)c * p.G]);
  for (int d = threadIdx.x; d < kD; d += blockDim.x) {
    float num = 0.f, den = 0.f;
    for (int c = 0; c < nch; ++c) {
      const float w = exp2f(p.part_lse[base + (long long)c * p.G] - M);
      den += w;
      num += w * p.part_o[(base + (long long)c * p.G) * kD + d];
    }
    p.out[((long long)b * p.Hq + h) * kD + d] = __float2bfloat16_rn(num / den);
  }
  if (threadIdx.x == 0) tstamp(p.trace2, 3);
}

// logical pages [n_blocks][page][d] -> DAK-PG swizzled pages (one thread per 16 bytes)
__global__ void pack_pages_kernel(const uint4* __restrict__ src, long long n_blocks, int page, uint4* __restrict__ dst) {
  const long long per_block = (long long)page * (kD / 8);
  const long long total = n_blocks * per_block;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / per_block;
    const int w = (int)(i % per_block);
    const int t = w / (kD / 8), j = w % (kD / 8);
    dst[blk * per_block + pg_off(t, j) / 16] = src[i];
  }
}

// append one token's K and V rows per (request, kv head) at position pos[b] (decode KV write)
__global__ void append_kernel(const uint4* __restrict__ k_new, const uint4* __restrict__ v_new, long long stride16,
                              const int* block_table, const int* pos, int B, int Hkv, int page, int max_pages,
                              uint4* k_hbm, uint4* v_hbm, uint4* k_host, uint4* v_host, unsigned long long* tr) {
  if (threadIdx.x == 0) tstamp(tr, 0);
  grid_dep_launch();
  grid_dep_wait();
  if (threadIdx.x == 0) tstamp(tr, 3);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (b, g, j)
  const int per = Hkv * (kD / 8);
  if (i >= B * per) return;
  const int b = i / per, g = (i % per) / (kD / 8), j = i % (kD / 8);
  const long long src = b * stride16 + (i % per);  // request rows may be strided (fused QKV output)
  const int ps = pos[b];
  const uint32_t e = (uint32_t)block_table[(long long)b * max_pages + ps / page];
  const long long idx = (long long)(e & ~kHostBit);
  const bool eh = (e & kHostBit) != 0;
  const int t = ps % page;
  const long long off = ((idx * Hkv + g) * (long long)page * kD * 2 + pg_off(t, j)) / 16;
  (eh ? k_host : k_hbm)[off] = k_new[src];
  (eh ? v_host : v_hbm)[off] = v_new[src];
}

// ------------------------------------------------------------------------------------ host side
static inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

struct Plan {
  Params p;
  int grid, smem;
  size_t ws_o, ws_lse;
};

static int g_sms = 0;

static dak_status make_plan(const dak_attention_args* a, Plan* out, bool need_ptrs) {
  if (!a) return fail(DAK_EINVAL, "dak_attention: args NULL");
  if (a->B <= 0 || a->Hq <= 0 || a->Hkv <= 0 || a->page_size <= 0 || a->max_pages <= 0 || a->chunk_pages <= 0)
    return fail(DAK_EINVAL, "dak_attention: sizes must be positive");
  if (a->Hq % a->Hkv) return fail(DAK_EINVAL, "dak_attention: Hq %% Hkv != 0");
  if (a->d != kD) return fail(DAK_EUNSUPPORTED, "dak_attention: head dim %d (this build: d = 128)", a->d);
  const int G = a->Hq / a->Hkv;
  if (G > kGmax) return fail(DAK_EUNSUPPORTED, "dak_attention: %d q heads per kv head > %d", G, kGmax);
  if (a->page_size % 16 || a->page_size > 256) return fail(DAK_EUNSUPPORTED, "dak_attention: page_size must be a multiple of 16, <= 256");
  const int max_chunks = (int)cdiv(a->max_pages, a->chunk_pages);
  if ((long long)a->B * max_chunks > kMaxPairs)
    return fail(DAK_EUNSUPPORTED, "dak_attention: B*ceil(max_pages/chunk_pages) = %lld > %d (raise chunk_pages)",
                (long long)a->B * max_chunks, kMaxPairs);
  Params p{};
  p.q = (const __nv_bfloat16*)a->q;
  p.out = (__nv_bfloat16*)a->out;
  p.k_hbm = (const char*)a->k_hbm;
  p.v_hbm = (const char*)a->v_hbm;
  p.k_host = (const char*)a->k_host;
  p.v_host = (const char*)a->v_host;
  p.block_table = a->block_table;
  p.seq_lens = a->seq_lens;
  p.B = a->B; p.Hq = a->Hq; p.Hkv = a->Hkv; p.G = G;
  p.q_stride = a->q_row_stride > 0 ? a->q_row_stride : (long long)a->Hq * kD;
  if (p.q_stride % 8) return fail(DAK_EINVAL, "dak_attention: q_row_stride must be a multiple of 8");
  p.page = a->page_size; p.max_pages = a->max_pages; p.chunk_pages = a->chunk_pages; p.max_chunks = max_chunks;
  const float scale = a->scale > 0.f ? a->scale : 1.0f / sqrtf((float)kD);
  p.scale_log2 = scale * 1.4426950408889634f;
  const size_t n_units = (size_t)a->B * a->Hkv * max_chunks;
  out->ws_o = n_units * G * kD * sizeof(float);
  out->ws_lse = n_units * G * sizeof(float);
  const dak_launch_cfg& c = a->cfg;
  p.stage_bytes = 2 * a->page_size * kD * 2;
  // SMEM: [1024 B barriers][ring: stages x (K page + V page)][q rows][merge scratch][pair prefix]
  const int scratch = kConsumerWarps * (kGmax * kD + 2 * kGmax) * 4;
  const int fixed = 1024 + scratch + a->B * max_chunks * 4;
  int max_stages = std::min((kSmemBudget - fixed) / (p.stage_bytes + kGmax * kD * 2), kMaxStages);
  if (max_stages < 2) return fail(DAK_EUNSUPPORTED, "dak_attention: page of %d B does not fit twice", p.stage_bytes / 2);
  int stages = c.stages > 0 ? std::min(c.stages, max_stages) : std::min(max_stages, 4);
  p.stages = std::max(2, stages);
  // host CTAs: one CTA keeps ~the link's saturating in-flight volume (calibration); window caps it
  int n_host = c.n_cta_host > 0 ? c.n_cta_host : 1;
  if (!a->k_host) n_host = 0;
  int window = p.stages;
  if (c.window > 0) window = std::min(c.window, p.stages);
  else if (c.congestion_control)
    window = std::max(1, std::min(p.stages, (int)cdiv(192 * 1024, (long long)p.stage_bytes * std::max(1, n_host))));
  p.window = window;
  int n_hbm = c.n_cta_hbm;
  if (n_hbm <= 0) {
    if (g_sms <= 0) {
      int dev = 0;
      DAK_CUDA_TRY(cudaGetDevice(&dev));
      DAK_CUDA_TRY(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    n_hbm = std::max(1, g_sms - n_host);
  }
  p.n_host = n_host;
  p.n_hbm = n_hbm;
  out->grid = n_host + n_hbm;
  p.off_q = 1024 + p.stages * p.stage_bytes;
  p.off_scratch = p.off_q + p.stages * kGmax * kD * 2;
  p.off_pairs = p.off_scratch + scratch;
  out->smem = p.off_pairs + a->B * max_chunks * 4;
  if (out->smem > kSmemBudget) return fail(DAK_EUNSUPPORTED, "dak_attention: shared memory plan %d B too large", out->smem);
  if (need_ptrs) {
    if (!a->q || !a->out || !a->block_table || !a->seq_lens) return fail(DAK_EINVAL, "dak_attention: NULL tensor");
    if (!a->k_hbm && !a->k_host) return fail(DAK_EINVAL, "dak_attention: no KV pool");
    if (!aligned16(a->q) || !aligned16(a->k_hbm) || !aligned16(a->v_hbm) || !aligned16(a->k_host) || !aligned16(a->v_host))
      return fail(DAK_EINVAL, "dak_attention: q and pools must be 16-byte aligned");
    if (!a->workspace || a->workspace_bytes < out->ws_o + out->ws_lse)
      return fail(DAK_EINVAL, "dak_attention: workspace too small (%zu < %zu)", a->workspace_bytes, out->ws_o + out->ws_lse);
    p.part_o = (float*)a->workspace;
    p.part_lse = (float*)((char*)a->workspace + out->ws_o);
  }
  out->p = p;
  return DAK_OK;
}

}  // namespace attn
}  // namespace dak

using namespace dak;

extern "C" {

dak_status dak_attention_workspace_size(const dak_attention_args* args, size_t* bytes) {
  if (!bytes) return fail(DAK_EINVAL, "dak_attention_workspace_size: bytes NULL");
  attn::Plan pl;
  dak_attention_args a = *args;
  if (a.cfg.n_cta_hbm <= 0) a.cfg.n_cta_hbm = 1;  // pure query: CTA count does not change the size
  dak_status st = attn::make_plan(&a, &pl, false);
  if (st != DAK_OK) return st;
  *bytes = pl.ws_o + pl.ws_lse;
  return DAK_OK;
}

dak_status dak_attention(const dak_attention_args* args, dak_stream_t stream) {
  attn::Plan pl;
  dak_status st = attn::make_plan(args, &pl, true);
  if (st != DAK_OK) return st;
  static int smem_set = 0;
  if (!smem_set) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(attn::split_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmemBudget));
    smem_set = 1;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = args->cfg.pdl ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(attn::kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pl.p.trace = trace_slot(DAK_KIND_ATTENTION, args->B, args->Hkv, pl.grid);
  const bool need_combine = pl.p.max_chunks > 1;
  pl.p.trace2 = need_combine ? trace_slot(DAK_KIND_COMBINE, args->B, args->Hq, args->B * args->Hq) : nullptr;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn::split_attention_kernel, pl.p));
  if (!need_combine) return DAK_OK;
  cudaLaunchConfig_t c2{};
  c2.gridDim = dim3(args->B * args->Hq);
  c2.blockDim = dim3(attn::kD);
  c2.dynamicSmemBytes = 0;
  c2.stream = (cudaStream_t)stream;
  c2.attrs = attr;
  c2.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&c2, attn::combine_kernel, pl.p));
  return DAK_OK;
}

dak_status dak_pack_kv_pages(const void* src, int64_t n_blocks, int32_t page_size, int32_t d, void* dst, dak_stream_t stream) {
  if (!src || !dst || n_blocks < 0) return fail(DAK_EINVAL, "dak_pack_kv_pages: bad arguments");
  if (d != attn::kD) return fail(DAK_EUNSUPPORTED, "dak_pack_kv_pages: d must be 128");
  if (page_size <= 0 || page_size % 16) return fail(DAK_EINVAL, "dak_pack_kv_pages: page_size must be a multiple of 16");
  if (!aligned16(src) || !aligned16(dst)) return fail(DAK_EINVAL, "dak_pack_kv_pages: pointers must be 16-byte aligned");
  if (n_blocks == 0) return DAK_OK;
  const long long total = n_blocks * (long long)page_size * (attn::kD / 8);
  const long long blocks = std::min<long long>(attn::cdiv(total, 256), 148LL * 64);
  attn::pack_pages_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, n_blocks, page_size, (uint4*)dst);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

dak_status dak_kv_append(const void* k_new, const void* v_new, int64_t row_stride, const int32_t* block_table,
                         const int32_t* positions, int32_t B, int32_t Hkv, int32_t d, int32_t page_size, int32_t max_pages,
                         void* k_hbm, void* v_hbm, void* k_host, void* v_host, int32_t pdl, dak_stream_t stream) {
  if (!k_new || !v_new || !block_table || !positions || B <= 0 || Hkv <= 0 || page_size <= 0 || max_pages <= 0)
    return fail(DAK_EINVAL, "dak_kv_append: bad arguments");
  if (d != attn::kD) return fail(DAK_EUNSUPPORTED, "dak_kv_append: d must be 128");
  const long long stride = row_stride > 0 ? row_stride : (long long)Hkv * d;
  if (stride % 8 || !aligned16(k_new) || !aligned16(v_new))
    return fail(DAK_EINVAL, "dak_kv_append: rows must be 16-byte aligned");
  const int n = B * Hkv * (attn::kD / 8);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn::append_kernel, (const uint4*)k_new, (const uint4*)v_new, stride / 8,
                                  block_table, positions, B, Hkv, page_size, max_pages, (uint4*)k_hbm, (uint4*)v_hbm,
                                  (uint4*)k_host, (uint4*)v_host, trace_slot(DAK_KIND_APPEND, B, Hkv, (n + 255) / 256)));
  return DAK_OK;
}

}  // extern "C"
