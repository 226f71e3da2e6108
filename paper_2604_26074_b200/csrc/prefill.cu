// dak_prefill_attention -- causal prefill attention over the HBM / host-split paged KV cache
// (§3.2: prefill attention has arithmetic intensity O(L) and is
// compute-bound at long L, which is the regime where the planner's Phase 2 can move up to
// B_h * T_comp bytes of an op to the host at no cost, P:L429 / P:L453).
//
// Work split: CTA = (request b, kv head g, block of 128 query rows), a query row being one (new
// token i, q head of g's GQA group) pair -- the G heads of a group share every K / V tile, so one
// CTA reads each tile once for all of them. Warps 0-7 each own 16 query rows (FlashAttention-2
// style, mma.sync m16n8k16 -> fp32: S = Q K^T in bf16 with K rows via ldmatrix, online softmax in
// the exp2 domain in registers, O += P V in fp16 with P re-used from the S accumulators as the A
// operand and V via ldmatrix.trans, the V tile converted bf16 -> fp16 in shared memory once per
// CTA by a convert warp (exact for |v| <= 65504, saturating beyond; reading R20 of DESIGN.md)); warp 8 lane 0 streams 64-token K and V tiles of the CTA's causal key range
// [0, kmax) into a ring of shared-memory stages with 1-D bulk copies (cp.async.bulk), each tile from
// the tier its page's block-table entry names (bit 31: host pool over the link, else HBM).
// Tiles are consumed in key order: the reduction order of a row depends on (seq_len, T) only, never
// on the tier split (bitwise r-invariant). DAK-PG pages (include/dak.h): row t's 16-byte chunks are
// swizzled by t & 7, so both ldmatrix forms are bank-conflict free.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "common.h"
#include "ptx.cuh"

namespace dak {
namespace pf {

using namespace ptx;

constexpr int kD = 128;
constexpr int kConsumers = 8;
constexpr int kThreads = (kConsumers + 2) * 32;  // + producer warp + V-convert warp
constexpr int kRows = kConsumers * 16;  // query rows per CTA
constexpr int kTile = 64;               // keys per stage
constexpr int kTileBytes = kTile * kD * 2;
constexpr int kMaxStages = 6;
constexpr uint32_t kHostBit = 0x80000000u;
constexpr int kListBytes = kThreads * 8 + 128;  // streamer scan list + per-warp counts

struct Params {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  const char* k_hbm;
  const char* v_hbm;
  const char* k_host;
  const char* v_host;
  const int* block_table;
  const int* seq_lens;
  int B, T, Hq, Hkv, G, page, max_pages;
  int blocks_per_bg;  // CTAs per (request, kv head)
  int stages;
  // host-tier streaming (workspace given): CTAs [0, n_stream) copy every host page of the batch once
  // over the link into the device staging pool (newest pages first) and raise its flag; compute
  // CTAs read host-tier tiles from the staging pool after the flag (no read amplification)
  int n_stream;
  char* k_stage;
  char* v_stage;
  int* flags;  // [B][Hkv][max_pages]
  float scale_log2;
  unsigned long long* trace;
  // tcgen05 form: K pools [0 HBM, 1 host, 2 staging], V pools [3, 4, 5] as 3-D tensors (64 elements,
  // 2 row halves, pool rows), box (64, 1, 64), no swizzle (DAK-PG rows are swizzled already)
  alignas(64) CUtensorMap kvmap[6];
};

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 4 + k] = t;
  }
}

// ---- host-tier streamer CTAs (blockIdx < n_stream; an SM reads one tier): every host page
// (b, g, page) of the batch is read ONCE over the link into the device staging pool, in the order
// the compute CTAs consume them -- (b, g) in grid order, newest page first within each -- so the
// first waves' pages arrive at the full link rate; each page's flag is raised with a release store.
// The scan over (b, g, page) runs on all threads, one item per thread per round, compacted in
// order through `list` (blockDim entries); the host items are dealt round-robin over the streamers
// and thread 0 keeps `slots` pages (K + V, 2 * page bytes each, in `ring`) in flight.
__device__ void stream_host_pages(const Params& p, unsigned char* ring, int slots, uint64_t* full, uint2* list) {
  const int nth = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* wsum = reinterpret_cast<int*>(list + nth);  // [32] per-warp host-item counts
  const int page_bytes = p.page * kD * 2;
  if (tid == 0) {
    for (int s = 0; s < slots; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_items = p.max_pages * p.B * p.Hkv;
  int seen = 0;                    // host items before this round (all threads)
  int issued = 0, done = 0;        // thread 0
  int qb[4], qg[4], qp[4];         // thread 0: the item in each slot
  auto complete = [&]() {          // thread 0: oldest slot landed -> staging pool, flag up
    const int sl = done % slots;
    mbar_wait(&full[sl], (uint32_t)((done / slots) & 1));
    const long long so = (((long long)qb[sl] * p.Hkv + qg[sl]) * p.max_pages + qp[sl]) * page_bytes;
    const unsigned char* src = ring + (size_t)sl * 2 * page_bytes;
    bulk_s2g(p.k_stage + so, src, page_bytes);
    bulk_s2g(p.v_stage + so, src + page_bytes, page_bytes);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    int* f = p.flags + ((long long)qb[sl] * p.Hkv + qg[sl]) * p.max_pages + qp[sl];
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
    ++done;
  };
  for (int k0 = 0; k0 < n_items; k0 += nth) {
    const int k = k0 + tid;
    uint32_t e = 0;
    bool host = false;
    if (k < n_items) {
      const int pg = p.max_pages - 1 - k % p.max_pages;
      const int b2 = k / p.max_pages / p.Hkv;
      if (pg < (p.seq_lens[b2] + p.page - 1) / p.page) {
        e = (uint32_t)p.block_table[(long long)b2 * p.max_pages + pg];
        host = (e & kHostBit) != 0;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, host);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, total = 0;
    for (int w = 0; w < (nth >> 5); ++w) {
      off += w < warp ? wsum[w] : 0;
      total += wsum[w];
    }
    if (host) list[off + __popc(bal & ((1u << lane) - 1u))] = make_uint2((uint32_t)k, e);
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < total; ++j) {
        if ((seen + j) % p.n_stream != (int)blockIdx.x) continue;
        if (issued - done == slots) complete();
        const int kk = (int)list[j].x;
        const uint32_t ee = list[j].y;
        const int sl = issued % slots;
        const int bg2 = kk / p.max_pages, g2 = bg2 % p.Hkv;
        const long long hoff = ((long long)(ee & ~kHostBit) * p.Hkv + g2) * page_bytes;
        unsigned char* dst = ring + (size_t)sl * 2 * page_bytes;
        mbar_expect_tx(&full[sl], 2u * page_bytes);
        bulk_g2s(dst, p.k_host + hoff, page_bytes, &full[sl]);
        bulk_g2s(dst + page_bytes, p.v_host + hoff, page_bytes, &full[sl]);
        qb[sl] = bg2 / p.Hkv;
        qg[sl] = g2;
        qp[sl] = p.max_pages - 1 - kk % p.max_pages;
        ++issued;
      }
    }
    seen += total;
    __syncthreads();  // list / wsum reused
  }
  if (tid == 0)
    while (done < issued) complete();
}

__global__ void __launch_bounds__(kThreads, 1) prefill_attention_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* vready = empty + kMaxStages;  // V tile of the slot converted to fp16 in place
  unsigned char* ring = smem + 1024;  // [stages][K tile | V tile]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages;
  const int page_bytes = p.page * kD * 2;
  if ((int)blockIdx.x < p.n_stream) {  // ---- host-tier streamer
    const int slots = min(4, S * kTileBytes / page_bytes);  // ring: S stages of 2 tiles
    stream_host_pages(p, ring, slots, full, reinterpret_cast<uint2*>(ring + (size_t)S * 2 * kTileBytes));
    return;
  }
  const int cta = (int)blockIdx.x - p.n_stream;
  const int bg = cta / p.blocks_per_bg, blk = cta % p.blocks_per_bg;
  const int b = bg / p.Hkv, g = bg % p.Hkv;
  const int L = p.seq_lens[b];
  const int rows = p.T * p.G;            // query rows of (b, g): row r = (token r / G, head r % G)
  const int r0 = blk * kRows;
  const int r_last = min(rows, r0 + kRows) - 1;
  const int kmax = L - p.T + r_last / p.G + 1;  // keys [0, kmax) cover every row of the block
  const int ntiles = (kmax + kTile - 1) / kTile;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
      mbar_init(&vready[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tstamp(p.trace, 0);
  }
  __syncthreads();

  if (warp == kConsumers) {  // ---- producer: K and V tile of every key block, newest keys first
    if (lane == 0) {
      const int* bt = p.block_table + (long long)b * p.max_pages;
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < ntiles; ++i) {
        if (i >= S) mbar_wait(&empty[s], ph ^ 1u);
        const int key0 = (ntiles - 1 - i) * kTile;
        const int pg = key0 / p.page;
        const uint32_t e = (uint32_t)bt[pg];
        const bool host = (e & kHostBit) != 0;
        const long long in_page = (long long)(key0 % p.page) * kD * 2;
        const char* ksrc = (host ? p.k_host : p.k_hbm) + ((long long)(e & ~kHostBit) * p.Hkv + g) * page_bytes + in_page;
        const char* vsrc = (host ? p.v_host : p.v_hbm) + ((long long)(e & ~kHostBit) * p.Hkv + g) * page_bytes + in_page;
        if (host && p.n_stream > 0) {  // staged copy once its flag is up (bounded wait: else read the link)
          const long long so = (((long long)b * p.Hkv + g) * p.max_pages + pg) * page_bytes + in_page;
          const int* f = p.flags + ((long long)b * p.Hkv + g) * p.max_pages + pg;
          int ready = 0;
          for (int it = 0; it < (1 << 22) && !ready; ++it) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(ready) : "l"(f) : "memory");
            if (!ready) __nanosleep(64);
          }
          if (ready) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            ksrc = p.k_stage + so;
            vsrc = p.v_stage + so;
          }
        }
        unsigned char* dst = ring + (size_t)s * 2 * kTileBytes;
        mbar_expect_tx(&full[s], 2u * kTileBytes);
        bulk_g2s(dst, ksrc, kTileBytes, &full[s]);
        bulk_g2s(dst + kTileBytes, vsrc, kTileBytes, &full[s]);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }

  if (warp == kConsumers + 1) {  // ---- V tiles bf16 -> fp16 in place, once per CTA (P V runs in fp16)
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < ntiles; ++i) {
      mbar_wait(&full[s], ph);
      uint4* v = reinterpret_cast<uint4*>(ring + (size_t)s * 2 * kTileBytes + kTileBytes);
#pragma unroll 4
      for (int c = lane; c < kTileBytes / 16; c += 32) {
        uint4 u = v[c];
        u.x = bf2_to_h2(u.x); u.y = bf2_to_h2(u.y); u.z = bf2_to_h2(u.z); u.w = bf2_to_h2(u.w);
        v[c] = u;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&vready[s]);
      if (++s == S) { s = 0; ph ^= 1u; }
    }
    return;
  }

  // ---- consumers: rows rw0 .. rw0 + 15 of the block
  const int gq = lane >> 2, cq = lane & 3;
  const int rw0 = r0 + warp * 16;
  const int ra = rw0 + gq, rb = rw0 + gq + 8;  // the two rows this thread holds
  // key limit of each row (causal): key k visible iff k < lim
  const int lim_a = ra < rows ? L - p.T + ra / p.G + 1 : 0;
  const int lim_b = rb < rows ? L - p.T + rb / p.G + 1 : 0;
  // Q as the A operand (rows ra / rb, 16 columns per k-step), straight from global memory
  uint32_t qa[kD / 16][4];
  {
    auto qrow = [&](int r) -> const uint32_t* {
      const int i = r / p.G, hh = r % p.G;
      return reinterpret_cast<const uint32_t*>(p.q + (((long long)b * p.T + i) * p.Hq + (long long)g * p.G + hh) * kD);
    };
    const uint32_t* qa_row = ra < rows ? qrow(ra) : nullptr;
    const uint32_t* qb_row = rb < rows ? qrow(rb) : nullptr;
#pragma unroll
    for (int ks = 0; ks < kD / 16; ++ks) {
      qa[ks][0] = qa_row ? qa_row[8 * ks + cq] : 0u;
      qa[ks][1] = qb_row ? qb_row[8 * ks + cq] : 0u;
      qa[ks][2] = qa_row ? qa_row[8 * ks + 4 + cq] : 0u;
      qa[ks][3] = qb_row ? qb_row[8 * ks + 4 + cq] : 0u;
    }
  }
  float o[kD / 8][4];
#pragma unroll
  for (int i = 0; i < kD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const int warp_lim = min(rows, rw0 + 16) > rw0 ? L - p.T + (min(rows, rw0 + 16) - 1) / p.G + 1 : 0;

  int s = 0;
  uint32_t ph = 0;
  for (int t = 0; t < ntiles; ++t) {
    mbar_wait(&full[s], ph);
    const int key0 = (ntiles - 1 - t) * kTile;  // newest keys first (the host prefix streams meanwhile)
    if (key0 < warp_lim) {  // tiles past every row of this warp only need the release below
      const uint32_t kb = su32(ring + (size_t)s * 2 * kTileBytes);
      const uint32_t vb = kb + kTileBytes;
      // ---- S = Q K^T : 16 rows x 64 keys (8 n8 tiles)
      float sc[kTile / 8][4];
#pragma unroll
      for (int j = 0; j < kTile / 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < kD / 16; ++ks) {
#pragma unroll
        for (int jj = 0; jj < kTile / 16; ++jj) {
          const int mtx = lane >> 3;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + pg_off(16 * jj + ((mtx >> 1) << 3) + (lane & 7), 2 * ks + (mtx & 1)), b0, b1, b2, b3);
          mma_bf16(sc[2 * jj], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
          mma_bf16(sc[2 * jj + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
        }
      }
      // ---- causal mask, scale, online softmax (exp2 domain); row a: sc[.][0..1], row b: sc[.][2..3]
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int j = 0; j < kTile / 8; ++j) {
        const int k = key0 + 8 * j + 2 * cq;
        sc[j][0] = k < lim_a ? sc[j][0] * p.scale_log2 : -INFINITY;
        sc[j][1] = k + 1 < lim_a ? sc[j][1] * p.scale_log2 : -INFINITY;
        sc[j][2] = k < lim_b ? sc[j][2] * p.scale_log2 : -INFINITY;
        sc[j][3] = k + 1 < lim_b ? sc[j][3] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, fmaxf(sc[j][0], sc[j][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[j][2], sc[j][3]));
      }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
      // rows with no visible key yet (or padding rows) keep m = -inf: use 0 as the reference
      const float ref0 = mn0 == -INFINITY ? 0.f : mn0, ref1 = mn1 == -INFINITY ? 0.f : mn1;
      const float al0 = exp2f(m[0] - ref0), al1 = exp2f(m[1] - ref1);
      m[0] = mn0;
      m[1] = mn1;
      float ls0 = 0.f, ls1 = 0.f;
      uint32_t pa[kTile / 16][4];  // P as the A operand of P V: k16 block kk = n8 tiles 2kk, 2kk+1
#pragma unroll
      for (int j = 0; j < kTile / 8; ++j) {
        const float p0 = exp2f(sc[j][0] - ref0), p1 = exp2f(sc[j][1] - ref0);
        const float p2 = exp2f(sc[j][2] - ref1), p3 = exp2f(sc[j][3] - ref1);
        // P in fp16 (11-bit significand, p in [0, 1]): bf16's 8 bits put up to 2^-9 relative error
        // on each weight, which for a row with a few dominant keys moves o by ~1% of |V| (measured
        // against the float64 oracle); the normaliser sums the same rounded weights
        const uint32_t h01 = pack_f16(p0, p1), h23 = pack_f16(p2, p3);
        const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&h01));
        const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&h23));
        ls0 += f01.x + f01.y;
        ls1 += f23.x + f23.y;
        pa[j >> 1][(j & 1) * 2 + 0] = h01;
        pa[j >> 1][(j & 1) * 2 + 1] = h23;
      }
      l[0] = l[0] * al0 + ls0;
      l[1] = l[1] * al1 + ls1;
#pragma unroll
      for (int i = 0; i < kD / 8; ++i) {
        o[i][0] *= al0; o[i][1] *= al0; o[i][2] *= al1; o[i][3] *= al1;
      }
      // ---- O += P V : V rows [key][d] (fp16 after the convert warp) through ldmatrix.trans
      mbar_wait(&vready[s], ph);
#pragma unroll
      for (int kk = 0; kk < kTile / 16; ++kk) {
#pragma unroll
        for (int i = 0; i < kD / 8; i += 2) {
          const int mtx = lane >> 3;
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + pg_off(16 * kk + ((mtx & 1) << 3) + (lane & 7), i + (mtx >> 1)), b0, b1, b2, b3);
          mma_f16(o[i], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
          mma_f16(o[i + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; ph ^= 1u; }
  }
  // ---- normalise and store: row sums over the 4 lanes of a row group
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    l[0] += __shfl_xor_sync(0xffffffffu, l[0], off);
    l[1] += __shfl_xor_sync(0xffffffffu, l[1], off);
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = half ? rb : ra;
    if (r >= rows) continue;
    const float inv = 1.f / l[half];
    const int i = r / p.G, hh = r % p.G;
    __nv_bfloat16* dst = p.out + (((long long)b * p.T + i) * p.Hq + (long long)g * p.G + hh) * kD;
#pragma unroll
    for (int n = 0; n < kD / 8; ++n)
      *reinterpret_cast<uint32_t*>(dst + 8 * n + 2 * cq) = pack_bf16(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
  }
  if (p.trace) {
    asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
    if (threadIdx.x == 0) tstamp(p.trace, 3);
  }
}


// ================================================================================================
// tcgen05 form (5th-gen tensor cores, TMEM accumulators). Same work split, host staging and
// newest-keys-first order as prefill_attention_kernel; the contractions run as
//   S[128 rows x 64 keys]  = Q[128 x 128 d] . K_tile^T   (8 x M128 N64 K16; A = Q from TMEM)
//   O_h[128 rows x 128 d] += P[128 x 32 keys] . V_half   (fp16: 2 x M128 N128 K16 per half; A = P from TMEM)
// Q (stored once) and P (written by the softmax warps with tcgen05.st) are A operands in tensor
// memory, so shared memory carries only the K / V tiles: the TMA writes (32 KB per tile), the V
// fp16 conversion (16 + 16 KB) and the tensor core's K / V reads (32 KB) -- with Q and P there too
// it moved 160 KB per tile, more than the MMAs' 512 cycles at ~128 B/clk.
// The K / V tiles come straight from the DAK-PG pages by TMA into canonical SWIZZLE_128B operands:
// a DAK-PG row is [d 0..63 | d 64..127] with the 16-byte chunks of each half already XOR-swizzled by
// row & 7, so a 3-D tensor map (64 elements, rows, 2 halves) with box (64, 64, 2) copies each half of
// 64 rows verbatim into an 8 KB block that IS the 128-byte-swizzled layout: K blocks are the K-major
// B operand of S (rows = keys), V blocks the MN-major B operand of P V (rows = keys, N = d; LBO =
// the 8 KB block stride, SBO = 1 KB per 8 keys). No transpose; V is converted bf16 -> fp16 in
// place (reading R20, as the mma.sync form; tcgen05 kind::f16 takes one type for A and B) by 4
// convert warps while S runs.
// Softmax: 8 warps, two per TMEM lane quadrant (thread = query row); warp parity c takes the tiles
// t = c mod 2 and keeps its OWN running max m_c, sum l_c and accumulator O_c (TMEM columns
// 128 (1 + c); P V of tile t accumulates into O_(t & 1)), so the two warps of a row never
// synchronise per tile and run half a period apart on their SM sub-partition (one's exponentials
// overlap the other's TMEM loads, barrier waits and stores -- the ping-pong FA4 gets from two
// query tiles). Merged once in the epilogue: O = (a_0 O_0 + a_1 O_1) / (a_0 l_0 + a_1 l_1),
// a_c = 2^(m_c - max m) (the log-sum-exp merge the split decode attention's combine kernel uses).
// exp2 domain, LAZY rescaling (m_c moves only when the tile max exceeds it by more than 8, then O_c
// is rescaled in TMEM; P <= 2^8), P in fp16 (tcgen05.st into TMEM), l_c summed from the fp32 P.
// The MMA warp waits on two barriers per tile: p_full(t) (softmax(t) has read S(t) and written
// P(t)) releases S(t + 2), issued first, then P V(t); vconv(t + 2) (tile landed, V converted).
// Warps: 0 producer (one lane issues), 1 MMA issuer (one elected lane), 2-5 V convert, 6-13
// softmax + epilogue.
constexpr int kUThreads = 14 * 32;
constexpr int kUStages = 6;
constexpr int kUOffStage = 1024;                             // stages: [K0 | K1 | V0 | V1] x 8 KB
constexpr int kUOffX = kUOffStage + kUStages * 2 * kTileBytes;  // epilogue m / l exchange; streamer list
constexpr int kUSmem = kUOffX + 4096 + 1024;                 // + alignment slack
// TMEM columns: S(t & 1) at 64 (t & 1), O_h at 128 (1 + h), Q (A operand, bf16 pairs) at 384,
// P(t & 1) (A operand, fp16 pairs) at 448 + 32 (t & 1)
constexpr uint32_t kTmO = 128, kTmQ = 384, kTmP = 448;

__global__ void __launch_bounds__(kUThreads, 1) prefill_umma_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint64_t* full = bars;                   // [kUStages] K / V tile landed (TMA tx)
  uint64_t* empty = bars + kUStages;       // [kUStages] P V of the stage's tile done (MMA commit)
  uint64_t* vconv = bars + 2 * kUStages;   // [kUStages] V converted to fp16 (4 convert warps)
  uint64_t* s_full = bars + 3 * kUStages;  // [2] S computed (MMA commit)
  uint64_t* p_full = s_full + 4;           // [2] P(t) of parity t & 1 written, O rescaled (4 warps)
  uint64_t* pv_done = s_full + 6;          // [2] P V of the parity's latest tile complete (MMA commit)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 512);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int page_bytes = p.page * kD * 2;
  if ((int)blockIdx.x < p.n_stream) {  // ---- host-tier streamer
    const int slots = min(4, kUStages * kTileBytes / page_bytes);  // the stage area
    stream_host_pages(p, smem + kUOffStage, slots, full, reinterpret_cast<uint2*>(smem + kUOffX));
    return;
  }
  const int cta = (int)blockIdx.x - p.n_stream;
  const int bg = cta / p.blocks_per_bg;
  const int blk = p.blocks_per_bg - 1 - cta % p.blocks_per_bg;  // longest causal ranges first (smaller tail)
  const int b = bg / p.Hkv, g = bg % p.Hkv;
  const int L = p.seq_lens[b];
  const int rows = p.T * p.G;
  const int r0 = blk * kRows;
  const int r_last = min(rows, r0 + kRows) - 1;
  const int kmax = L - p.T + r_last / p.G + 1;
  const int nt = (kmax + kTile - 1) / kTile;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kUStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&vconv[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tstamp(p.trace, 0);
  }
  if (warp == 1) {  // TMEM: all 512 columns (see kTmO / kTmQ / kTmP)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0)
    for (int i = 0; i < 6; ++i) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.kvmap[i])) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp >= 6) {  // ---- Q -> TMEM (A operand of S): thread = row, warp half h = d [64 h, 64 h + 64)
    const int q4 = warp & 3, h = (warp - 6) >> 2;
    const int r = 32 * q4 + lane, gr = r0 + r;
    uint32_t v[32];
    if (gr < rows) {
      const int i = gr / p.G, hh = gr % p.G;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (((long long)b * p.T + i) * p.Hq + (long long)g * p.G + hh) * kD + 64 * h);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 u = src[j];
        v[4 * j] = u.x; v[4 * j + 1] = u.y; v[4 * j + 2] = u.z; v[4 * j + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0u;
    }
    const uint32_t qa = tmem + ((uint32_t)(32 * q4) << 16) + kTmQ + 32u * (uint32_t)h;
    tmem_st16(qa, v);
    tmem_st16(qa + 16u, v + 16);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {  // ---- producer: K / V tiles by TMA, newest keys first (lane 0 issues)
    const int* bt = p.block_table + (long long)b * p.max_pages;
    const int* fl = p.flags + ((long long)b * p.Hkv + g) * p.max_pages;
    int ready_until = -1;  // staged host tiles up to here are known to have their flag up
    // block-table entries of tiles [w0, w0 + 32) in lane t - w0 (one load per 32 tiles, the next
    // window's load in flight while this one is used: a dependent global load per tile would pace
    // the whole pipeline)
    auto bt_of = [&](int tl) -> uint32_t { return tl < nt ? (uint32_t)bt[(nt - 1 - tl) * kTile / p.page] : 0u; };
    // lane i of the window also holds tile w0 + i's page, key offset in the page and staging-pool
    // row, so a tile costs three shuffles (no integer divisions on the producer's critical path)
    int pg_w = 0, ip_w = 0, rs_w = 0;
    auto win_geom = [&](int tl) {
      const int key0 = (nt - 1 - min(tl, nt - 1)) * kTile;
      pg_w = key0 / p.page;
      ip_w = key0 - pg_w * p.page;
      rs_w = (((b * p.Hkv + g) * p.max_pages) + pg_w) * p.page + ip_w;
    };
    uint32_t e_win = bt_of(lane), e_next = bt_of(32 + lane);
    win_geom(lane);
    int rp_w = (int)(e_win & ~kHostBit) * p.Hkv * p.page + g * p.page + ip_w;  // HBM / host pool row
    for (int t = 0; t < nt; ++t) {
      const int s2 = t % kUStages;
      if (t > 0 && (t & 31) == 0) {
        e_win = e_next;
        e_next = bt_of(t + 32 + lane);
        win_geom(t + lane);
        rp_w = (int)(e_win & ~kHostBit) * p.Hkv * p.page + g * p.page + ip_w;
      }
      const uint32_t e = __shfl_sync(0xffffffffu, e_win, t & 31);
      const bool host = (e & kHostBit) != 0;
      int tier = host ? 1 : 0;
      int row = __shfl_sync(0xffffffffu, rp_w, t & 31);  // pool row of the tile's first key
      const int row_stage = __shfl_sync(0xffffffffu, rs_w, t & 31);
      const int pg = __shfl_sync(0xffffffffu, pg_w, t & 31);
      if (host && p.n_stream > 0) {
        if (t > ready_until) {
          // the warp polls the flags of tiles t .. t + 31 at once (acquire), until tile t's is up
          // (bounded: after it, tile t is read over the link directly -- the same bits)
          const int tl = t + lane;
          bool mine = true;  // tiles past the end or in HBM count as ready
          if (tl < nt) {
            const int pgl = (nt - 1 - tl) * kTile / p.page;
            if (bt_of(tl) & kHostBit) {
              int f = 0;
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(fl + pgl) : "memory");
              mine = f != 0;
            }
          }
          uint32_t mask = __ballot_sync(0xffffffffu, mine);
          for (int it = 0; it < (1 << 22) && !(mask & 1u); ++it) {
            __nanosleep(64);
            int f = 1;
            if (lane == 0) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(fl + pg) : "memory");
            mask = __ballot_sync(0xffffffffu, lane == 0 && f != 0);
          }
          if (mask & 1u) {
            ready_until = t + (~mask ? __ffs(~mask) - 1 : 32) - 1;
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        if (t <= ready_until) {
          tier = 2;
          row = row_stage;
        }
      }
      if (lane == 0) {
        if (t >= kUStages) mbar_wait(&empty[s2], (uint32_t)((t / kUStages - 1) & 1));
        unsigned char* dst = smem + kUOffStage + (size_t)s2 * 2 * kTileBytes;
        const uint64_t km = reinterpret_cast<uint64_t>(&p.kvmap[tier]), vm = reinterpret_cast<uint64_t>(&p.kvmap[3 + tier]);
        mbar_expect_tx(&full[s2], 2u * kTileBytes);
        tma_3d(dst, km, 0, (int)row, 0, &full[s2]);          // K: [half][64 rows][128 B]
        tma_3d(dst + 16384, vm, 0, (int)row, 0, &full[s2]);  // V
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // ---- MMA issuer
    // instruction descriptors: f32 accumulate, M = 128; S: bf16 x bf16, N = 64, both K-major;
    // P V: f16 x f16, N = 128, B (V) MN-major (bit 16)
    const uint32_t id_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t id_o = (1u << 4) | (1u << 16) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t st_u = su32(smem + kUOffStage);
    uint32_t leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
    auto issue_s = [&](int t) {  // S[t & 1] = Q . K_t^T (tile t landed and its V converted)
      const int s2 = t % kUStages;
      mbar_wait(&vconv[s2], (uint32_t)((t / kUStages) & 1));
      tc_fence_after();
      if (leader) {
        const uint32_t kb = st_u + (uint32_t)s2 * 2 * kTileBytes;
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks)  // A = Q from TMEM: 8 columns (16 bf16) per K step
          umma_ts(tmem + (uint32_t)((t & 1) * 64), tmem + kTmQ + 8u * ks,
                  umma_desc_sw128(kb + (ks >> 2) * 8192 + (ks & 3) * 32), id_s, ks != 0);
        umma_commit(&s_full[t & 1]);
      }
      __syncwarp();
    };
    issue_s(0);
    if (nt > 1) issue_s(1);
    for (int t = 0; t < nt; ++t) {
      const int bb = t & 1, s2 = t % kUStages;
      // softmax(t) done: S buffer bb has been read (S(t + 2) may overwrite it) and P(t) is written;
      // V(t) was converted before S(t) was issued
      mbar_wait(&p_full[bb], (uint32_t)((t >> 1) & 1));
      tc_fence_after();
      if (t + 2 < nt) issue_s(t + 2);  // first: softmax(t + 2) waits for it
      if (leader) {  // O_bb += P(t) V(t): the tiles of parity bb accumulate in their own O
        const uint32_t vb = st_u + (uint32_t)s2 * 2 * kTileBytes + 16384;
#pragma unroll
        for (int ks = 0; ks < kTile / 16; ++ks)  // A = P from TMEM: 8 columns (16 fp16) per K step
          umma_ts(tmem + kTmO + 128u * bb, tmem + kTmP + 32u * bb + 8u * ks,
                  umma_desc_sw128_mn(vb + ks * 2048, 8192), id_o, ((t >> 1) | ks) != 0);
        umma_commit(&empty[s2]);    // K / V stage free
        umma_commit(&pv_done[bb]);  // P(t) consumed; O_bb holds tiles <= t of its parity
      }
      __syncwarp();
    }
  } else if (warp >= 2 && warp <= 5) {  // ---- V: bf16 -> fp16 in place (16 KB per tile)
    const int tt = threadIdx.x - 64;  // 0..127
    for (int t = 0; t < nt; ++t) {
      const int s2 = t % kUStages;
      mbar_wait(&full[s2], (uint32_t)((t / kUStages) & 1));
      unsigned char* v = smem + kUOffStage + (size_t)s2 * 2 * kTileBytes + 16384;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint4* w = reinterpret_cast<uint4*>(v) + tt + 128 * i;
        uint4 u = *w;
        u.x = bf2_to_h2(u.x); u.y = bf2_to_h2(u.y); u.z = bf2_to_h2(u.z); u.w = bf2_to_h2(u.w);
        *w = u;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&vconv[s2]);
    }
  } else {  // ---- softmax warps 6..13: thread = query row, warp parity c = the tiles t = c mod 2
    const int q4 = warp & 3, c = (warp - 6) >> 2;
    const int r = 32 * q4 + lane;  // row of the block (TMEM lane)
    const int gr = r0 + r;
    const int lim = gr < rows ? L - p.T + gr / p.G + 1 : 0;  // keys [0, lim) visible
    const int lim_w = __reduce_min_sync(0xffffffffu, (unsigned)lim);  // tiles below it need no mask
    const uint32_t lane_base = (uint32_t)(32 * q4) << 16;
    const uint32_t o_c = tmem + lane_base + kTmO + 128u * (uint32_t)c;  // this parity's O accumulator
    const uint32_t s_c = tmem + lane_base + 64u * (uint32_t)c;          // S buffer of this parity
    const uint32_t p_c = tmem + lane_base + kTmP + 32u * (uint32_t)c;   // P buffer of this parity
    float m = -INFINITY, l = 0.f;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    for (int t = c, k = 0; t < nt; t += 2, ++k) {  // k: this warp's k-th tile (barrier phase k & 1)
      const int key0 = (nt - 1 - t) * kTile;
      mbar_wait(&s_full[c], (uint32_t)(k & 1));
      tc_fence_after();
      uint32_t sv_u[kTile];
#pragma unroll
      for (int c0 = 0; c0 < kTile; c0 += 16) tmem_ld16(s_c + (uint32_t)c0, sv_u + c0);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < kTile; ++j) asm volatile("" : "+r"(sv_u[j]));  // keep every use after the wait
      float* sv = reinterpret_cast<float*>(sv_u);
      if (key0 + kTile > lim_w) {  // the warp's diagonal tiles: mask keys >= lim
#pragma unroll
        for (int j = 0; j < kTile; ++j) sv[j] = key0 + j < lim ? sv[j] : -INFINITY;
      }
      float mq[4];  // 4 independent max chains
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* x = sv + 16 * j;
        float a = fmax3(x[0], x[1], x[2]), b2 = fmax3(x[3], x[4], x[5]);
        a = fmax3(a, x[6], x[7]);
        b2 = fmax3(b2, x[8], x[9]);
        a = fmax3(a, x[10], x[11]);
        b2 = fmax3(b2, x[12], x[13]);
        mq[j] = fmax3(a, b2, fmaxf(x[14], x[15]));
      }
      const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * p.scale_log2;  // scale > 0
      // the P V of this parity's previous tile must be complete before its P buffer is rewritten
      // and before its O is rescaled
      if (k > 0) mbar_wait(&pv_done[c], (uint32_t)((k - 1) & 1));
      // lazy reference max: move it (and rescale O, l) only when the tile max exceeds it by > 8
      const bool move = mx > m + 8.f;
      if (__any_sync(0xffffffffu, move)) {
        const float m_new = move ? mx : m;
        const float alpha = m == -INFINITY ? 0.f : ex2_ftz(m - m_new);  // 1 for rows that keep m
        if (k > 0 && __any_sync(0xffffffffu, move && m != -INFINITY)) {
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < kD; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(o_c + (uint32_t)c0, v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
            tmem_st16(o_c + (uint32_t)c0, v);
          }
        }
        l *= alpha;
        m = m_new;
      }
      const float ref = m == -INFINITY ? 0.f : m;
      const float2 nref2 = make_float2(-ref, -ref);
      float2 l2 = make_float2(0.f, 0.f), l3 = make_float2(0.f, 0.f);
      uint32_t pw[kTile / 2];  // P as fp16 pairs -> TMEM (A operand of P V)
#pragma unroll
      for (int e = 0; e < kTile / 2; ++e) {
        float2 x = ffma2(make_float2(sv[2 * e], sv[2 * e + 1]), sc2, nref2);
        x.x = ex2_ftz(x.x);
        x.y = ex2_ftz(x.y);
        pw[e] = pack_f16(x.x, x.y);
        if (e & 1) l3 = fadd2(l3, x); else l2 = fadd2(l2, x);
      }
      tmem_st16(p_c, pw);
      tmem_st16(p_c + 16u, pw + 16);
      l += (l2.x + l2.y) + (l3.x + l3.y);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[c]);
    }
    // ---- epilogue: merge the parities, O = (a_0 O_0 + a_1 O_1) / (a_0 l_0 + a_1 l_1), a_c = 2^(m_c - M);
    // this warp writes d [64 c, 64 c + 64). An O never written (nt == 1: parity 1 has no tile) has
    // a_c = 0 and is not read.
    float* xch = reinterpret_cast<float*>(smem + kUOffX);  // [m | l][2 parities][128 rows]
    xch[c * 128 + r] = m;
    xch[256 + c * 128 + r] = l;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q4) : "memory");
    const float m0 = c ? xch[r] : m, m1 = c ? m : xch[128 + r];
    const float l0 = c ? xch[256 + r] : l, l1 = c ? l : xch[384 + r];
    const float M = fmaxf(m0, m1);
    const float a0 = m0 == -INFINITY ? 0.f : ex2_ftz(m0 - M), a1 = m1 == -INFINITY ? 0.f : ex2_ftz(m1 - M);
    const float lt = a0 * l0 + a1 * l1;
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const float s0 = a0 * inv, s1 = a1 * inv;
    const bool use1 = nt > 1;
    mbar_wait(&pv_done[(nt - 1) & 1], (uint32_t)(((nt - 1) >> 1) & 1));  // the last P V (covers both parities)
    tc_fence_after();
    __nv_bfloat16* dst = nullptr;
    if (gr < rows) {
      const int i = gr / p.G, hh = gr % p.G;
      dst = p.out + (((long long)b * p.T + i) * p.Hq + (long long)g * p.G + hh) * kD;
    }
#pragma unroll 1
    for (int c0 = 64 * c; c0 < 64 * c + 64; c0 += 16) {
      uint32_t v0[16], v1[16];
      tmem_ld16(tmem + lane_base + kTmO + (uint32_t)c0, v0);
      tmem_ld16(tmem + lane_base + kTmO + 128u + (uint32_t)c0, v1);
      tmem_wait_ld();
      if (dst) {
        float o[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) o[e] = __uint_as_float(v0[e]) * s0 + (use1 ? __uint_as_float(v1[e]) * s1 : 0.f);
        uint4 w0, w1;
        w0.x = pack_bf16(o[0], o[1]); w0.y = pack_bf16(o[2], o[3]); w0.z = pack_bf16(o[4], o[5]); w0.w = pack_bf16(o[6], o[7]);
        w1.x = pack_bf16(o[8], o[9]); w1.y = pack_bf16(o[10], o[11]); w1.z = pack_bf16(o[12], o[13]); w1.w = pack_bf16(o[14], o[15]);
        reinterpret_cast<uint4*>(dst + c0)[0] = w0;
        reinterpret_cast<uint4*>(dst + c0)[1] = w1;
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (threadIdx.x == 0) tstamp(p.trace, 3);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace pf
}  // namespace dak

using namespace dak;

// A K or V pool (HBM, host or staging) as a 3-D bf16 tensor: 64 elements (128 B), rows (stride
// 256 B; the pool's extent is not known here, so the row count is a bound, 2^30, that every
// in-range row index satisfies), 2 row halves (stride 128 B). A (64, 64, 2) box lands as two 8 KB
// blocks [half][row][64 elements].
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static dak_status encode_kv_map(CUtensorMap* m, const void* base) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* f = nullptr;
    DAK_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
    if (qr != cudaDriverEntryPointSuccess || !f) return fail(DAK_ECUDA, "dak_prefill_attention: cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)f;
  }
  const cuuint64_t dims[3] = {64, 1ull << 30, 2};
  const cuuint64_t strides[2] = {256, 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)pf::kTile, 2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DAK_ECUDA, "dak_prefill_attention: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DAK_OK;
}

extern "C" {

static dak_status prefill_plan(const dak_prefill_args* a, pf::Params* p, int* grid, int* smem) {
  if (!a) return fail(DAK_EINVAL, "dak_prefill_attention: args NULL");
  if (a->B <= 0 || a->T <= 0 || a->Hq <= 0 || a->Hkv <= 0 || a->page_size <= 0 || a->max_pages <= 0)
    return fail(DAK_EINVAL, "dak_prefill_attention: sizes must be positive");
  if (a->Hq % a->Hkv) return fail(DAK_EINVAL, "dak_prefill_attention: Hq %% Hkv != 0");
  if (a->d != pf::kD) return fail(DAK_EUNSUPPORTED, "dak_prefill_attention: head dim %d (this build: d = 128)", a->d);
  if (a->page_size % pf::kTile) return fail(DAK_EUNSUPPORTED, "dak_prefill_attention: page_size must be a multiple of 64");
  if (!a->q || !a->out || !a->block_table || !a->seq_lens || (!a->k_hbm && !a->k_host))
    return fail(DAK_EINVAL, "dak_prefill_attention: NULL tensor");
  if (!aligned16(a->q) || !aligned16(a->out) || !aligned16(a->k_hbm) || !aligned16(a->v_hbm) || !aligned16(a->k_host) ||
      !aligned16(a->v_host))
    return fail(DAK_EINVAL, "dak_prefill_attention: pointers must be 16-byte aligned");
  pf::Params q{};
  q.q = (const __nv_bfloat16*)a->q;
  q.out = (__nv_bfloat16*)a->out;
  q.k_hbm = (const char*)a->k_hbm;
  q.v_hbm = (const char*)a->v_hbm;
  q.k_host = (const char*)a->k_host;
  q.v_host = (const char*)a->v_host;
  q.block_table = a->block_table;
  q.seq_lens = a->seq_lens;
  q.B = a->B; q.T = a->T; q.Hq = a->Hq; q.Hkv = a->Hkv; q.G = a->Hq / a->Hkv;
  q.page = a->page_size; q.max_pages = a->max_pages;
  q.blocks_per_bg = (a->T * q.G + pf::kRows - 1) / pf::kRows;
  q.stages = a->cfg.stages > 0 ? std::min(a->cfg.stages, pf::kMaxStages) : pf::kMaxStages;
  if (q.stages < 2) q.stages = 2;
  const float scale = a->scale > 0.f ? a->scale : 1.0f / sqrtf((float)pf::kD);
  q.scale_log2 = scale * 1.4426950408889634f;
  // host-tier streaming through the caller's workspace: [flags][K stage][V stage]
  const size_t flag_bytes = ((size_t)a->B * a->Hkv * a->max_pages * 4 + 255) / 256 * 256;
  const size_t stage_bytes = (size_t)a->B * a->Hkv * a->max_pages * a->page_size * pf::kD * 2;
  q.n_stream = 0;
  if (a->workspace && a->k_host) {
    if (a->workspace_bytes < flag_bytes + 2 * stage_bytes || !aligned16(a->workspace))
      return fail(DAK_EINVAL, "dak_prefill_attention: workspace %zu < %zu", a->workspace_bytes, flag_bytes + 2 * stage_bytes);
    q.n_stream = a->cfg.n_cta_host > 0 ? a->cfg.n_cta_host : 4;
    q.flags = (int*)a->workspace;
    q.k_stage = (char*)a->workspace + flag_bytes;
    q.v_stage = q.k_stage + stage_bytes;
  }
  if (q.n_stream > 0) {  // a streamer slot holds one page of K and of V in the kernel's stage ring
    const long long ring = a->cfg.force_path == 2 ? (long long)q.stages * 2 * pf::kTileBytes : (long long)pf::kUStages * 2 * pf::kTileBytes;
    if (2LL * a->page_size * pf::kD * 2 > ring)
      return fail(DAK_EUNSUPPORTED, "dak_prefill_attention: page_size %d too large for host staging (ring %lld B)", a->page_size, ring);
  }
  const long long g = (long long)a->B * a->Hkv * q.blocks_per_bg + q.n_stream;
  if (g > 0x7fffffffLL) return fail(DAK_EUNSUPPORTED, "dak_prefill_attention: grid too large");
  if (a->cfg.force_path != 2) {
    const void* base[6] = {a->k_hbm, a->k_host, q.k_stage, a->v_hbm, a->v_host, q.v_stage};
    for (int i = 0; i < 6; ++i) {
      const void* ptr = base[i] ? base[i] : (a->k_hbm ? a->k_hbm : a->k_host);  // unused tier: any valid pointer
      const dak_status st = encode_kv_map(&q.kvmap[i], ptr);
      if (st != DAK_OK) return st;
    }
  }
  *p = q;
  *grid = (int)g;
  *smem = 1024 + q.stages * 2 * pf::kTileBytes + pf::kListBytes + 1024;
  return DAK_OK;
}

dak_status dak_prefill_workspace_size(const dak_prefill_args* a, size_t* bytes) {
  if (!a || !bytes || a->B <= 0 || a->Hkv <= 0 || a->max_pages <= 0 || a->page_size <= 0)
    return fail(DAK_EINVAL, "dak_prefill_workspace_size: bad arguments");
  const size_t flag_bytes = ((size_t)a->B * a->Hkv * a->max_pages * 4 + 255) / 256 * 256;
  *bytes = flag_bytes + 2 * (size_t)a->B * a->Hkv * a->max_pages * a->page_size * pf::kD * 2;
  return DAK_OK;
}

dak_status dak_prefill_attention(const dak_prefill_args* args, dak_stream_t stream) {
  pf::Params p;
  int grid = 0, smem = 0;
  dak_status st = prefill_plan(args, &p, &grid, &smem);
  if (st != DAK_OK) return st;
  static bool attr = false;
  if (!attr) {
    DAK_CUDA_TRY(cudaFuncSetAttribute(pf::prefill_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      1024 + pf::kMaxStages * 2 * pf::kTileBytes + pf::kListBytes + 1024));
    DAK_CUDA_TRY(cudaFuncSetAttribute(pf::prefill_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pf::kUSmem));
    attr = true;
  }
  const bool umma = args->cfg.force_path != 2;  // tcgen05 by default; force_path 2: the mma.sync form
  if (p.n_stream > 0)  // staged-page flags start lowered (a memset node under graph capture)
    DAK_CUDA_TRY(cudaMemsetAsync(p.flags, 0, (size_t)args->B * args->Hkv * args->max_pages * 4, (cudaStream_t)stream));
  p.trace = trace_slot(DAK_KIND_PREFILL, args->B, args->T, grid);
  if (umma)
    pf::prefill_umma_kernel<<<grid, pf::kUThreads, pf::kUSmem, (cudaStream_t)stream>>>(p);
  else
    pf::prefill_attention_kernel<<<grid, pf::kThreads, smem, (cudaStream_t)stream>>>(p);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

}  // extern "C"
