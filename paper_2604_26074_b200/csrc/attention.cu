// dak_attention — split paged GQA decode attention for sm_100a (PAPER §4, §3.1).
//
// The KV cache is paged; each page of one kv head is a [page_size, d] bf16 block living either in
// the HBM pool or in the pinned, device-mapped host pool (block-table bit 31 selects the tier).
// Work is split flash-decoding style into units (request b, kv head g, chunk c of chunk_pages
// pages). Each CTA reads exactly one tier: CTAs [0, n_host) take the units whose chunk
// starts on a host page, the rest take HBM units, round-robin by the unit's rank within its tier.
// Each unit is owned by ONE warp, which walks its tiles in order and is its own producer: lane 0
// streams the warp's next tiles (K and V rows of a page, 1-D bulk copies = TMA engine, completing on
// mbarriers) into a private SMEM ring whose depth the CTA sizes from the warps that own units; host
// CTAs cap their in-flight bytes (congestion control). The
// warp computes on tensor cores (mma.sync m16n8k16 bf16->fp32):
//   S^T[16 tokens x 8 heads] = K_tile . Q^T       (all q heads of the GQA group in one n8 tile)
//   online softmax per head (exp2 domain), P^T fed back as the B operand via movmatrix.trans
//   O^T[d x 8 heads]       += V_tile^T . P^T      (ldmatrix.trans on the swizzled V rows)
// and writes the normalised output directly (single-chunk request) or the chunk partial
// (o, log2-sum-exp) to workspace.
// A combine kernel merges the chunk partials of each (b, q-head) in chunk order -> bf16 output.
// Every reduction order is fixed by (seq_len, chunk_pages, page_size): outputs are independent
// of which pages live on the host (bitwise r-invariance).
//
// KV page layout ("DAK-PG"): a page of one kv head is [page_size][d] bf16 with the 16-byte chunk
// j of token row t stored at chunk ((j>>3)<<3) | ((j&7) ^ (t&7)) (bank-conflict-free ldmatrix).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "ptx.cuh"

namespace dak {
namespace attn {

using namespace ptx;

constexpr int kD = 128;
constexpr int kGmax = 8;              // q heads per kv head handled in one n8 tile
constexpr int kWarps = 8;              // each warp produces and consumes its own units
constexpr int kThreads = 32 * kWarps;
constexpr int kMaxSlots = 16;          // ring slots per warp
constexpr int kRingOff = 1152;         // barriers (1 KB) + unit count + scan scratch below the ring
constexpr int kMaxPairs = 8192;       // (request, chunk) pairs scheduled per launch
constexpr int kSmemBudget = 226 * 1024;  // 227 KB opt-in minus the 1 KB the extern alignment adds statically
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
  int n_host, n_hbm;
  int auto_host;      // 1: host-CTA count chosen in-kernel from the block table (cfg.n_cta_host == 0)
  int ring_bytes;     // SMEM ring bytes per CTA, shared by the CTA's active warps
  int max_slots;      // ring slots per warp cap (<= kMaxSlots)
  int host_window;    // host CTAs: max in-flight tiles per warp (0: none)
  int host_inflight;  // host CTAs: max in-flight bytes per CTA (congestion control; 0: none)
  int host_budget;    // host bytes in flight over all host CTAs (auto host-CTA count)
  int off_pairs;
  const uint4* k_new;  // fused append: new token rows (16-byte units), nullptr: off
  const uint4* v_new;
  long long new_stride16;  // 16-byte units between requests of k_new / v_new
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

// ------------------------------------------------------------------------------------ PTX glue: ptx.cuh

// Unit k of a tier -> (pair index, kv head). pref[p] = tier-matching pairs before pair p.
__device__ __forceinline__ int find_pair(const int* pref, int n_pairs, int rank) {
  int lo = 0, hi = n_pairs - 1;  // largest p with pref[p] <= rank and pair p matching
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= rank) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Work split: one WARP owns a whole unit (request b, kv head g, chunk c) and walks its tokens in
// order with the online softmax in registers -- no cross-warp merge, no CTA barrier per unit. Unit k
// of a tier goes to CTA (k mod n) and warp ((k div n) mod 8), so short contexts put up to 8 units in
// flight per SM. Each warp is its own producer: lane 0 keeps the warp's private ring of `slots`
// slots filled with the warp's next tiles (a slot = `tt` token rows of K and of V, 16 or 32,
// contiguous rows of a DAK-PG page: two bulk copies completing on the slot's mbarrier) and refills
// a slot as soon as the warp has consumed it. The ring depth is sized per CTA from the units it
// actually owns, so a CTA with few units keeps as many bytes in flight as one with eight (Little's
// law, not the unit count, sets the per-SM bandwidth). q of the unit's GQA group is read straight
// into the B-fragment registers.
__global__ void __launch_bounds__(kThreads, 1) split_attention_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);            // [8 warps][kMaxSlots]
  int* s_count = reinterpret_cast<int*>(full + kWarps * kMaxSlots);
  int* warp_tot = s_count + 4;                                     // [kWarps] scan scratch
  unsigned char* ring = smem + kRingOff;                          // [8 warps][slots][slot bytes]
  int* pref = reinterpret_cast<int*>(smem + p.off_pairs);       // [B * max_chunks] tier-rank prefix
  int* s_len = pref + p.B * p.max_chunks;                          // [B] seq_lens

  const int cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int page_bytes = p.page * kD * 2;

  // each warp's ring barriers, one per lane, by the warp itself (128 serial inits by one thread
  // sat on the kernel's pre-wait critical path)
  if (lane < kMaxSlots) mbar_init(&full[warp * kMaxSlots + lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (threadIdx.x == 0) tstamp(p.trace, 0);
  grid_dep_launch();
  const int n_pairs = p.B * p.max_chunks;
  // CTA roles (one tier per SM): given, or chosen below from the block table (auto)
  int n_host = p.n_host, n_hbm = p.n_hbm, host_inflight = p.host_inflight;
  // ---- schedule inputs, loaded ONCE with independent loads (two dependent rounds in all: seq_lens,
  // then the first block-table entry of every (request, chunk) pair); pref[i] holds the pair's flags
  // (bit 0: the chunk exists, bit 1: its first page is on the host) until the scan overwrites it
  for (int b = threadIdx.x; b < p.B; b += kThreads) s_len[b] = p.seq_lens[b];
  {
    // seq_lens and the first block-table entry of every pair are loaded together (the entry of a
    // chunk beyond the request's length is read but ignored: c * chunk_pages < max_pages always):
    // one round trip, not two
    int cnt = 0;
#pragma unroll 4
    for (int i = threadIdx.x; i < n_pairs; i += kThreads) {
      const int b = i / p.max_chunks, c = i - b * p.max_chunks;
      const int L = p.seq_lens[b];
      const uint32_t e = (uint32_t)p.block_table[(long long)b * p.max_pages + c * p.chunk_pages];
      const int npg = (L + p.page - 1) / p.page;
      int f = 0;
      if (c * p.chunk_pages < npg) {
        f = 1 | ((e & kHostBit) ? 2 : 0);
        cnt += f >> 1;
      }
      pref[i] = f;
    }
    if (p.auto_host) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0) warp_tot[warp] = cnt;
    }
    __syncthreads();
  }
  if (p.auto_host) {
    // one host CTA per 4 host units (request, kv head, chunk) -- host CTAs are bound by the link
    // latency, so a few keep more bytes in flight -- capped at 16 (congestion control),
    // none when the block table names no host chunk
    int hu = 0;
    for (int w = 0; w < kWarps; ++w) hu += warp_tot[w];
    __syncthreads();
    hu *= p.Hkv;
    n_host = hu ? min(min(16, (hu + 3) / 4), (int)gridDim.x - 1) : 0;
    n_hbm = (int)gridDim.x - n_host;
    if (host_inflight > 0 && n_host > 0) host_inflight = max(2 * 16 * kD * 2, p.host_budget / n_host);
  }
  const bool host = cta < n_host;
  const int my_j = host ? cta : cta - n_host;
  const int my_n = host ? n_host : n_hbm;
  // Block table and seq_lens are step inputs, and every KV row except the newest token's was
  // written by earlier steps: the schedule and those tiles do not wait for the previous kernel
  // (griddepcontrol.wait). q and the tile holding the new token (position seq_len - 1, written by
  // the KV-append kernel just before) are read only after it (ABI contract in dak.h).
  // ---- schedule: pairs (b, c) linearised p = b*max_chunks + c, tier-matching ones ranked (exclusive
  // prefix over the flags in SMEM, block-wide, fixed order)
  {
    int carry = 0;
    for (int base = 0; base < n_pairs; base += kThreads) {
      const int i = base + threadIdx.x;
      int f = 0;
      if (i < n_pairs) {
        const int fl = pref[i];
        f = (fl & 1) && (((fl >> 1) & 1) != 0) == host;
      }
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
      for (int w = 0; w < kWarps; ++w) tot += warp_tot[w];
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) *s_count = carry;
    __syncthreads();
  }
  const int n_units = *s_count * p.Hkv;
  const int stride = my_n * kWarps;  // units between consecutive units of one warp
  // ---- ring geometry of this CTA: warps that own a unit share the ring bytes
  const int my_units = my_j < n_units ? (n_units - my_j + my_n - 1) / my_n : 0;
  const int active = min(kWarps, my_units);
  if (warp >= active) return;
  const int per_warp = (p.ring_bytes / active) & ~127;
  // 32-token tiles (two 8 KB copies) whenever the page allows: measured faster than 16-token tiles
  // even at one slot per warp (eight warps interleave; the per-copy cost favours larger copies)
  const int tt = p.page % 32 == 0 ? 32 : 16;
  const int slot_bytes = 2 * tt * kD * 2;
  int slots = max(1, min(p.max_slots, per_warp / slot_bytes));
  if (host && p.host_window > 0) slots = min(slots, p.host_window);
  // congestion cap on in-flight host bytes, but never below double buffering per warp (one slot per
  // warp exposes the full link latency per tile: C4 B = 4 at r*, 0.90 -> 0.97 of EB(r*) without it)
  if (host && host_inflight > 0) slots = min(slots, max(2, host_inflight / (active * slot_bytes)));
  const int tile_bytes = tt * kD * 2;

  uint64_t* wf = full + warp * kMaxSlots;
  unsigned char* wr = ring + (size_t)warp * per_warp;

  // ---- producer cursor (lane 0 issues; every lane tracks it so the control flow stays uniform)
  int pk = my_j + warp * my_n, ptok = 0, pt1 = 0, pb = 0, pg = 0, pL = 0;
  int ppg = 0, pr0 = 0;  // cursor's page index within the request and row within the page
  auto unit_open = [&](int k, int& b, int& g, int& L, int& t0, int& t1) {
    const int pr = find_pair(pref, n_pairs, k / p.Hkv);
    g = k % p.Hkv;
    b = pr / p.max_chunks;
    const int c = pr % p.max_chunks;
    L = s_len[b];
    t0 = c * p.chunk_pages * p.page;
    t1 = min(L, t0 + p.chunk_pages * p.page);
  };
  // block-table entries of pages [ent_base, ent_base + 32) of the cursor's request, one per lane,
  // loaded one tile ahead of their first use so the load latency hides behind a tile of compute
  int ent = 0, ent_base = 0;
  auto load_ents = [&]() {
    ent_base = ppg;
    const int pgi = ent_base + lane;
    ent = pgi < p.max_pages ? p.block_table[(long long)pb * p.max_pages + pgi] : 0;
  };
  auto open_next = [&]() {
    unit_open(pk, pb, pg, pL, ptok, pt1);
    ppg = ptok / p.page;  // = chunk * chunk_pages
    pr0 = 0;
    load_ents();
  };
  if (pk < n_units) open_next();
  int pit = 0, ps = 0;  // tiles issued, slot of the next one (incremental: no divisions per tile)
  auto issue = [&]() {
    const int s = ps;
    const int r0 = pr0;
    const uint32_t e = (uint32_t)__shfl_sync(0xffffffffu, ent, ppg - ent_base);
    if (lane == 0) {
      const long long idx = (long long)(e & ~kHostBit);
      const bool eh = (e & kHostBit) != 0;
      const long long off = (idx * p.Hkv + pg) * (long long)page_bytes + (long long)r0 * kD * 2;
      unsigned char* dst = wr + (size_t)s * slot_bytes;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the slot
      mbar_expect_tx(&wf[s], 2u * tile_bytes);
      bulk_g2s(dst, (eh ? p.k_host : p.k_hbm) + off, tile_bytes, &wf[s]);
      bulk_g2s(dst + tile_bytes, (eh ? p.v_host : p.v_hbm) + off, tile_bytes, &wf[s]);
    }
    ++pit;
    if (++ps == slots) ps = 0;
    ptok += tt;
    pr0 += tt;
    if (pr0 == p.page) {  // tt divides page
      pr0 = 0;
      ++ppg;
    }
    if (ptok >= pt1) {
      pk += stride;
      if (pk < n_units) open_next();
    } else if (ppg - ent_base >= 32) {
      load_ents();
    }
  };
  // prologue: only tiles of old tokens (not holding position L - 1) before the dependency wait; with
  // the fused append every tile (the new token's row is patched into the slot after the wait)
  while (pit < slots && pk < n_units && (p.k_new || ptok + tt <= pL - 1)) issue();
  grid_dep_wait();
  if (threadIdx.x == 0) tstamp(p.trace, 1);
  while (pit < slots && pk < n_units) issue();

  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column pair
  int cs = 0;
  uint32_t cph = 0;  // consumer slot and its barrier phase
  bool first_unit = true;
  for (int k = my_j + warp * my_n; k < n_units; k += stride) {
    int b, g, L, t0, t1;
    unit_open(k, b, g, L, t0, t1);
    const int npg = (L + p.page - 1) / p.page;
    // q of the GQA group as the B operand: b0 = q[head gq][16 ks + 2 cq, +1], b1 = ... + 8 (heads >= G: 0)
    uint32_t qb[kD / 16][2];
    {
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(p.q + (long long)b * p.q_stride + ((long long)g * p.G + gq) * kD);
#pragma unroll
      for (int ks = 0; ks < kD / 16; ++ks) {
        qb[ks][0] = gq < p.G ? qrow[8 * ks + cq] : 0u;
        qb[ks][1] = gq < p.G ? qrow[8 * ks + 4 + cq] : 0u;
      }
    }
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    float o[kD / 16][4];
#pragma unroll
    for (int i = 0; i < kD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

    for (int tile0 = t0; tile0 < t1; tile0 += tt) {
      const int s = cs;
      mbar_wait(&wf[s], cph);
      if (++cs == slots) {
        cs = 0;
        cph ^= 1u;
      }
      const uint32_t kslot = su32(wr + (size_t)s * slot_bytes);
      if (p.k_new && tile0 <= L - 1 && L - 1 < tile0 + tt) {
        // fused KV append: the new token's K (lanes 0-15) / V (lanes 16-31) chunks go into this
        // slot's row (the page row is stale) and into the page for later steps
        const int t = L - 1 - tile0, j = lane & 15;
        const uint4 v = (lane < 16 ? p.k_new : p.v_new)[(long long)b * p.new_stride16 + (long long)g * (kD / 8) + j];
        const uint32_t off = (uint32_t)(t * (kD * 2) + ((((j >> 3) << 3) | ((j & 7) ^ (t & 7))) << 4));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(kslot + (lane < 16 ? 0u : (uint32_t)tile_bytes) + off),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the slot's next TMA refill
        const int pg_i = (L - 1) / p.page;
        const uint32_t e = (uint32_t)p.block_table[(long long)b * p.max_pages + pg_i];
        const long long idx = (long long)(e & ~kHostBit);
        const bool eh = (e & kHostBit) != 0;
        const char* pool = lane < 16 ? (eh ? p.k_host : p.k_hbm) : (eh ? p.v_host : p.v_hbm);
        *reinterpret_cast<uint4*>(const_cast<char*>(pool) + (idx * p.Hkv + g) * (long long)page_bytes +
                                  pg_off((L - 1) % p.page, j)) = v;
        __syncwarp();
      }
      // The tile's (up to two) 16-token sub-tiles are processed together: their S^T = K . Q^T chains
      // interleave, ONE online-softmax update (max, rescale of O) covers the whole tile, then
      // O^T += V^T . P^T for both. P enters the tensor core as bf16 hi + lo parts (p = hi + lo to
      // ~16 significant bits; V stays bf16: no per-tile conversion of V), l sums the same hi + lo.
      const int nsub = (min(tt, t1 - tile0) + 15) >> 4;  // sub-tiles holding a valid token (1 or 2)
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int ks = 0; ks < kD / 16; ++ks) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u < nsub) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(kslot + u * 16 * (kD * 2) + pg_off(lane & 15, 2 * ks + (lane >> 4)), a0, a1, a2, a3);
            mma_bf16(sc[u], a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
          }
        }
      }
      // ---- scale, mask, online softmax (exp2 domain), per head column, once per tile
      float sv[2][4];
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tok0 = tile0 + 16 * u;
        const bool v0 = u < nsub && tok0 + gq < t1, v1 = u < nsub && tok0 + gq + 8 < t1;
        sv[u][0] = v0 ? sc[u][0] * p.scale_log2 : -INFINITY;
        sv[u][1] = v0 ? sc[u][1] * p.scale_log2 : -INFINITY;
        sv[u][2] = v1 ? sc[u][2] * p.scale_log2 : -INFINITY;
        sv[u][3] = v1 ? sc[u][3] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, fmaxf(sv[u][0], sv[u][2]));
        mx1 = fmaxf(mx1, fmaxf(sv[u][1], sv[u][3]));
      }
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);  // finite: the tile has a valid token
      const float al0 = exp2f(m[0] - mn0), al1 = exp2f(m[1] - mn1);
      m[0] = mn0;
      m[1] = mn1;
      uint32_t ph[2][2], pl[2][2];  // [sub][rows gq | gq + 8] bf16x2 (head 2cq, 2cq + 1): hi and lo parts
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const float e0 = exp2f(sv[u][2 * r] - mn0), e1 = exp2f(sv[u][2 * r + 1] - mn1);
          const uint32_t hi = pack_bf16(e0, e1);
          const float h0 = __uint_as_float(hi << 16), h1 = __uint_as_float(hi & 0xffff0000u);
          const uint32_t lo = pack_bf16(e0 - h0, e1 - h1);
          ph[u][r] = hi;
          pl[u][r] = lo;
          ls0 += h0 + __uint_as_float(lo << 16);
          ls1 += h1 + __uint_as_float(lo & 0xffff0000u);
        }
      }
      l[0] = l[0] * al0 + ls0;
      l[1] = l[1] * al1 + ls1;
#pragma unroll
      for (int i = 0; i < kD / 16; ++i) {
        o[i][0] *= al0; o[i][1] *= al1; o[i][2] *= al0; o[i][3] *= al1;
      }
      // ---- O^T[d x heads] += V^T . P^T  (P^T as the B operand: transposed 8x8 blocks of P)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u < nsub) {
          const uint32_t bh0 = movm_t(ph[u][0]), bh1 = movm_t(ph[u][1]);
          const uint32_t bl0 = movm_t(pl[u][0]), bl1 = movm_t(pl[u][1]);
          const uint32_t vbase = kslot + tile_bytes + u * 16 * (kD * 2);
#pragma unroll
          for (int i = 0; i < kD / 16; ++i) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vbase + pg_off((lane & 7) + ((lane >> 4) << 3), 2 * i + ((lane >> 3) & 1)), a0, a1, a2, a3);
            mma_bf16(o[i], a0, a1, a2, a3, bh0, bh1);
            mma_bf16(o[i], a0, a1, a2, a3, bl0, bl1);
          }
        }
      }
      __syncwarp();
      if (pk < n_units) issue();  // refill the slot just consumed with the stream's next tile
    }
    // ---- l per head column: sum over the 8 lane groups holding the column
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l[0] += __shfl_xor_sync(0xffffffffu, l[0], off);
      l[1] += __shfl_xor_sync(0xffffffffu, l[1], off);
    }
    // lane holds O^T[d][head] for d = 16 i + gq (+8), head = 2 cq (+1)
    const bool direct = npg <= p.chunk_pages;  // the request is one chunk: no combine needed
    const int c = t0 / (p.chunk_pages * p.page);
    const long long ubase = (((long long)b * p.Hkv + g) * p.max_chunks + c) * p.G;
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
      const int hh = 2 * cq + hc;
      if (hh < p.G) {
        const float inv = 1.f / l[hc];
        if (direct) {
          __nv_bfloat16* dst = p.out + ((long long)b * p.Hq + g * p.G + hh) * kD;
#pragma unroll
          for (int i = 0; i < kD / 16; ++i) {
            dst[16 * i + gq] = __float2bfloat16_rn(o[i][hc] * inv);
            dst[16 * i + gq + 8] = __float2bfloat16_rn(o[i][2 + hc] * inv);
          }
        } else {
          float* dst = p.part_o + (ubase + hh) * kD;
#pragma unroll
          for (int i = 0; i < kD / 16; ++i) {
            dst[16 * i + gq] = o[i][hc] * inv;
            dst[16 * i + gq + 8] = o[i][2 + hc] * inv;
          }
          if (gq == 0) p.part_lse[ubase + hh] = m[hc] + log2f(l[hc]);
        }
      }
    }
    if (first_unit && lane == 0 && warp == 0) tstamp(p.trace, 2);  // first unit of warp 0 done
    first_unit = false;
  }
  if (p.trace) {
    asm volatile("bar.sync 1, %0;" ::"r"(active * 32) : "memory");
    if (lane == 0 && warp == 0) tstamp(p.trace, 3);
  }
}

// merge chunk partials: out[b, h, :] = sum_c w_c o_c / sum_c w_c, w_c = 2^(lse_c - max lse).
// One CTA of W warps per (b, q head): warp j accumulates chunks c = j, j + W, ... with a running
// max (lane = 4 dims, float4 loads, several chunks in flight), then the W warp partials are
// rescaled to the common max and summed in warp order. W = 4 when a request has <= 16 chunks (the
// decode steps' usual split: B * Hq CTAs fit one wave beside the attention kernel's; 16-warp CTAs
// took two waves at b64, 3.3 us from the attention's end to the last CTA's start), else 16 (one
// L2 round trip for 128 chunks). The order depends only on the chunk count and max_chunks
// (bitwise r-invariant).
template <int W>
__global__ void __launch_bounds__(W * 32) combine_kernel(const Params p) {
  __shared__ float s_red[W];
  __shared__ float4 s_acc[W][kD / 4];
  __shared__ float s_den[W];
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long base = (((long long)b * p.Hkv + g) * p.max_chunks) * p.G + hh;  // + c*G
  // warp j: running max m, den = sum 2^(lse_c - m), acc = sum 2^(lse_c - m) o_c over its chunks
  // (no separate max pass: the loads of every chunk are independent of the arithmetic)
  float m = -INFINITY, den = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
  for (int c = warp; c < nch; c += W) {
    const long long u = base + (long long)c * p.G;
    const float ls = p.part_lse[u];
    const float4 v = reinterpret_cast<const float4*>(p.part_o + u * kD)[lane];
    const float mn = fmaxf(m, ls);
    const float sc = exp2f(m - mn), w = exp2f(ls - mn);
    m = mn;
    den = den * sc + w;
    acc.x = acc.x * sc + w * v.x; acc.y = acc.y * sc + w * v.y;
    acc.z = acc.z * sc + w * v.z; acc.w = acc.w * sc + w * v.w;
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) {
    s_den[warp] = den;
    s_red[warp] = m;
  }
  __syncthreads();
  if (threadIdx.x < kD / 4) {
    const int nw = min(nch, W);  // warps that own a chunk
    float M = s_red[0];
    for (int w = 1; w < nw; ++w) M = fmaxf(M, s_red[w]);
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    float dn = 0.f;
    for (int w = 0; w < nw; ++w) {  // fixed warp order
      const float sc = exp2f(s_red[w] - M);
      const float4 v = s_acc[w][threadIdx.x];
      t.x += sc * v.x; t.y += sc * v.y; t.z += sc * v.z; t.w += sc * v.w;
      dn += sc * s_den[w];
    }
    const float inv = 1.f / dn;
    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(p.out + ((long long)b * p.Hq + h) * kD) + 2 * threadIdx.x;
    dst[0] = __floats2bfloat162_rn(t.x * inv, t.y * inv);
    dst[1] = __floats2bfloat162_rn(t.z * inv, t.w * inv);
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

// KV re-placement across decode steps (dak_kv_replace's moves): copy whole pages (all kv heads,
// K and V) from their old slot to their new slot. The DAK-PG layout is the same in both pools, so a
// page moves as raw 16-byte words. moves[2i] = old entry, moves[2i+1] = new entry (bit 31: host).
__global__ void migrate_pages_kernel(const int* __restrict__ moves, int n, long long page_u4, uint4* k_hbm,
                                     uint4* v_hbm, uint4* k_host, uint4* v_host) {
  const long long total = (long long)n * 2 * page_u4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / (2 * page_u4);
    const long long r = i - m * 2 * page_u4;
    const bool is_v = r >= page_u4;
    const long long w = is_v ? r - page_u4 : r;
    const uint32_t src = (uint32_t)moves[2 * m], dst = (uint32_t)moves[2 * m + 1];
    const uint4* sp = (src & kHostBit) ? (is_v ? v_host : k_host) : (is_v ? v_hbm : k_hbm);
    uint4* dp = (dst & kHostBit) ? (is_v ? v_host : k_host) : (is_v ? v_hbm : k_hbm);
    dp[(long long)(dst & ~kHostBit) * page_u4 + w] = sp[(long long)(src & ~kHostBit) * page_u4 + w];
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

// Llama decode KV write with rotary positions: rotate q (in place) and k of the new token of every
// request at positions[b] (rotate-half pairs (i, i + d/2), angle pos / theta^(2i/d), computed in
// double then fp32 sincos of the reduced angle), then append k (rotated) and v to the page pools.
// One 64-thread CTA per (request b, head hh) of the [q heads | k heads | v heads] row; thread i owns
// the rotate-half pair (i, i + 64). With part != nullptr the two values are first reduced from the
// producing linear's split-K fp32 partials: bf16(sum_s part[s][b][c]) in split order (the split-K
// reduce, fused here; part row stride = (Hq + 2 Hkv) * d, B rows per split). q and k heads are
// rotated (angle pos / theta^(2i/d), double-reduced, fp32 sincos); k and v heads are also written
// into the page at position pos (DAK-PG swizzle). The row in qkv is rewritten (q is read by attention).
__global__ void __launch_bounds__(64) rope_append_kernel(__nv_bfloat16* qkv, long long stride, int Hq, int Hkv,
                                                         const int* pos, double log2_theta, const int* block_table,
                                                         int page, int max_pages, uint4* k_hbm, uint4* v_hbm,
                                                         uint4* k_host, uint4* v_host, unsigned long long* tr,
                                                         const float* part, int S, int B) {
  if (threadIdx.x == 0) tstamp(tr, 0);
  grid_dep_launch();
  const int H3 = Hq + 2 * Hkv;
  const int b = blockIdx.x / H3, hh = blockIdx.x % H3;
  const int i = threadIdx.x;  // 0 .. 63
  // positions and the block table are step inputs (not written by the previous kernel): their
  // loads overlap the dependency wait
  const int ps = pos[b];
  const uint32_t e = hh >= Hq ? (uint32_t)block_table[(long long)b * max_pages + ps / page] : 0u;
  grid_dep_wait();
  __nv_bfloat16* v = qkv + (long long)b * stride + (long long)hh * kD;
  float x1, x2;
  if (part) {
    const long long cols = (long long)H3 * kD, split = (long long)B * cols;
    const float* pr = part + (long long)b * cols + (long long)hh * kD;
    // all S partials are loaded before the (fixed-order) sum: one L2 round trip, not S
    float v1[16], v2[16];
#pragma unroll
    for (int sp = 0; sp < 16; ++sp) {
      if (sp < S) {
        v1[sp] = __ldcg(pr + sp * split + i);
        v2[sp] = __ldcg(pr + sp * split + i + kD / 2);
      }
    }
    float a1 = v1[0], a2 = v2[0];
#pragma unroll
    for (int sp = 1; sp < 16; ++sp) {
      if (sp < S) {
        a1 += v1[sp];
        a2 += v2[sp];
      }
    }
    for (int sp = 16; sp < S; ++sp) {  // (more than 16 splits: the rest one by one, same order)
      a1 += pr[sp * split + i];
      a2 += pr[sp * split + i + kD / 2];
    }
    x1 = __bfloat162float(__float2bfloat16_rn(a1));
    x2 = __bfloat162float(__float2bfloat16_rn(a2));
  } else {
    x1 = __bfloat162float(v[i]);
    x2 = __bfloat162float(v[i + kD / 2]);
  }
  __nv_bfloat16 o1 = __float2bfloat16_rn(x1), o2 = __float2bfloat16_rn(x2);
  if (hh < Hq + Hkv) {  // rotary on q and k heads
    const double inv = exp2(-(2.0 * i / kD) * log2_theta);
    const double ang = fmod((double)ps * inv, 6.283185307179586476925286766559);
    float sn, cs;
    sincosf((float)ang, &sn, &cs);
    o1 = __float2bfloat16_rn(x1 * cs - x2 * sn);
    o2 = __float2bfloat16_rn(x2 * cs + x1 * sn);
  }
  v[i] = o1;
  v[i + kD / 2] = o2;
  if (hh >= Hq) {  // k or v head: append at position ps
    const bool is_k = hh < Hq + Hkv;
    const int g = is_k ? hh - Hq : hh - Hq - Hkv;
    const long long idx = (long long)(e & ~kHostBit);
    const bool eh = (e & kHostBit) != 0;
    const int t = ps % page;
    char* pool = reinterpret_cast<char*>(is_k ? (eh ? k_host : k_hbm) : (eh ? v_host : v_hbm));
    char* pg = pool + (idx * Hkv + g) * (long long)page * kD * 2;
    *reinterpret_cast<__nv_bfloat16*>(pg + pg_off(t, i >> 3) + (i & 7) * 2) = o1;
    *reinterpret_cast<__nv_bfloat16*>(pg + pg_off(t, (i + kD / 2) >> 3) + (i & 7) * 2) = o2;
  }
  if (threadIdx.x == 0) tstamp(tr, 3);
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
  // per warp: a ring of tile slots [K tt rows][V tt rows]; the kernel sizes tt and the slot count
  // per CTA from the warps that own units (the ring bytes are shared by them)
  p.off_pairs = kSmemBudget - (a->B * max_chunks + a->B) * 4;
  p.off_pairs &= ~127;
  p.ring_bytes = p.off_pairs - kRingOff;
  if (p.ring_bytes < kWarps * 2 * 16 * kD * 2)
    return fail(DAK_EUNSUPPORTED, "dak_attention: tile ring does not fit (B * chunks too large)");
  p.max_slots = c.stages > 0 ? std::min(c.stages, kMaxSlots) : kMaxSlots;
  // host CTAs (caller-sized: ~one per 8 host units, i.e. one unit per warp; default 2). Congestion
  // control caps the host bytes in flight: 512 KB over all host CTAs keeps the PCIe link
  // saturated with 8 KB copies (256 KB reached only ~42 GB/s at C4 B = 4, r*) without queueing more
  // host CTAs: caller-sized, or (n_cta_host == 0) chosen in-kernel from the block table
  p.auto_host = c.n_cta_host <= 0 && a->k_host != nullptr;
  int n_host = c.n_cta_host > 0 ? c.n_cta_host : (a->k_host ? 1 : 0);
  if (!a->k_host) n_host = 0;
  p.host_window = c.window > 0 ? c.window : 0;
  // congestion budget: host bytes in flight over all host CTAs (dak_calibrate, else 512 KB)
  p.host_budget = c.host_inflight_kb > 0 ? c.host_inflight_kb * 1024 : 512 * 1024;
  p.host_inflight = (c.window <= 0 && c.congestion_control) ? (int)std::max<long long>(2 * 16 * kD * 2, p.host_budget / std::max(1, n_host)) : 0;
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
  out->smem = p.off_pairs + (a->B * max_chunks + a->B) * 4;
  if (need_ptrs) {
    if (!a->q || !a->out || !a->block_table || !a->seq_lens) return fail(DAK_EINVAL, "dak_attention: NULL tensor");
    if (!a->k_hbm && !a->k_host) return fail(DAK_EINVAL, "dak_attention: no KV pool");
    if ((a->k_new == nullptr) != (a->v_new == nullptr)) return fail(DAK_EINVAL, "dak_attention: k_new and v_new go together");
    if (a->k_new) {
      const long long st = a->kv_new_stride > 0 ? a->kv_new_stride : (long long)a->Hkv * kD;
      if (st % 8 || !aligned16(a->k_new) || !aligned16(a->v_new))
        return fail(DAK_EINVAL, "dak_attention: k_new / v_new rows must be 16-byte aligned");
      p.k_new = (const uint4*)a->k_new;
      p.v_new = (const uint4*)a->v_new;
      p.new_stride16 = st / 8;
    }
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
  const bool small = pl.p.max_chunks <= 16;
  c2.blockDim = dim3(small ? 4 * 32 : 16 * 32);
  c2.dynamicSmemBytes = 0;
  c2.stream = (cudaStream_t)stream;
  c2.attrs = attr;
  c2.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&c2, small ? attn::combine_kernel<4> : attn::combine_kernel<16>, pl.p));
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

dak_status dak_kv_migrate(const int32_t* moves, int32_t n_moves, int32_t Hkv, int32_t page_size, int32_t d, void* k_hbm,
                          void* v_hbm, void* k_host, void* v_host, dak_stream_t stream) {
  if (n_moves < 0 || (n_moves > 0 && !moves) || Hkv <= 0 || page_size <= 0 || d <= 0 || (d * 2) % 16)
    return fail(DAK_EINVAL, "dak_kv_migrate: bad arguments");
  if (n_moves == 0) return DAK_OK;
  if (!aligned16(k_hbm) || !aligned16(v_hbm) || !aligned16(k_host) || !aligned16(v_host))
    return fail(DAK_EINVAL, "dak_kv_migrate: pools must be 16-byte aligned");
  const long long page_u4 = (long long)Hkv * page_size * d * 2 / 16;
  const long long total = (long long)n_moves * 2 * page_u4;
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 4096);
  attn::migrate_pages_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(moves, n_moves, page_u4, (uint4*)k_hbm, (uint4*)v_hbm,
                                                                       (uint4*)k_host, (uint4*)v_host);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

dak_status dak_rope_kv_append(void* qkv, int64_t row_stride, int32_t B, int32_t Hq, int32_t Hkv, int32_t d,
                             const int32_t* positions, float rope_theta, const int32_t* block_table, int32_t page_size,
                             int32_t max_pages, void* k_hbm, void* v_hbm, void* k_host, void* v_host, int32_t pdl,
                             dak_stream_t stream) {
  return dak::rope_kv_append_part(qkv, row_stride, B, Hq, Hkv, d, positions, rope_theta, block_table, page_size,
                                  max_pages, k_hbm, v_hbm, k_host, v_host, pdl, stream, nullptr, 1);
}

}  // extern "C"

dak_status dak::rope_kv_append_part(void* qkv, int64_t row_stride, int32_t B, int32_t Hq, int32_t Hkv, int32_t d,
                                    const int32_t* positions, float rope_theta, const int32_t* block_table,
                                    int32_t page_size, int32_t max_pages, void* k_hbm, void* v_hbm, void* k_host,
                                    void* v_host, int32_t pdl, void* stream, const float* part, int32_t S) {
  if (!qkv || !positions || !block_table || B <= 0 || Hq <= 0 || Hkv <= 0 || page_size <= 0 || max_pages <= 0 ||
      !(rope_theta > 1.f))
    return fail(DAK_EINVAL, "dak_rope_kv_append: bad arguments");
  if (d != attn::kD) return fail(DAK_EUNSUPPORTED, "dak_rope_kv_append: d must be 128");
  const long long stride = row_stride > 0 ? row_stride : (long long)(Hq + 2 * Hkv) * d;
  if (stride < (long long)(Hq + 2 * Hkv) * d || stride % 8 || !aligned16(qkv))
    return fail(DAK_EINVAL, "dak_rope_kv_append: qkv rows must be 16-byte aligned and hold q, k, v");
  if (part && (!aligned16(part) || S < 1)) return fail(DAK_EINVAL, "dak_rope_kv_append: bad split-K partials");
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(B * (Hq + 2 * Hkv));
  cfg.blockDim = dim3(64);
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAK_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn::rope_append_kernel, (__nv_bfloat16*)qkv, stride, Hq, Hkv, positions,
                                  (double)log2((double)rope_theta), block_table, page_size, max_pages, (uint4*)k_hbm,
                                  (uint4*)v_hbm, (uint4*)k_host, (uint4*)v_host,
                                  trace_slot(DAK_KIND_APPEND, B, Hkv, B * (Hq + 2 * Hkv)), part, (int)S, (int)B));
  return DAK_OK;
}

