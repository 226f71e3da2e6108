// Planner inputs and placement on the host side of the C ABI:
//   dak_global_offload_bytes -- capacity -> global host budget Y_req and R (§3.2, P:L757,
//                               P:L981)
//   dak_decode_ops           -- the per-op profile of one decode step: C_i, units, FLOPs, T_i
//                               (P:L383-388, P:L422 footnote, P:L981 footnote)
//   dak_kv_place             -- the KV byte partition of one attention op: oldest split-KV chunks
//                               on the host, chunk-major across requests (
//                               DESIGN.md readings R7, R15)
//   dak_kv_replace           -- that partition moved along as the requests grow across decode
//                               steps (reading R23)
//   dak_calib_select         -- the choice of the congestion-control operating point from the
//                               calibration sweep (reading R24)
// Compiled with -ffp-contract=off: every double below is one IEEE rounding in the written order,
// so the T_i values are bit-identical to the oracle's definition (oracle/models.py decode_ops),
// which the CPU tests check. The oracle is never linked or called from here.
#include <algorithm>
#include <vector>

#include "common.h"

namespace {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

extern "C" {

dak_status dak_global_offload_bytes(int64_t weight_bytes, int64_t kv_bytes, int64_t hbm_budget_bytes,
                                    int64_t host_capacity_bytes, int64_t* y_req_bytes, double* ratio) {
  if (!y_req_bytes) return dak::fail(DAK_EINVAL, "dak_global_offload_bytes: y_req_bytes NULL");
  if (weight_bytes < 0 || kv_bytes < 0 || hbm_budget_bytes < 0)
    return dak::fail(DAK_EINVAL, "dak_global_offload_bytes: negative size");
  const int64_t footprint = weight_bytes + kv_bytes;
  const int64_t over = footprint - hbm_budget_bytes;
  // the overflow must fit the host tier
  if (host_capacity_bytes >= 0 && over > host_capacity_bytes)
    return dak::fail(DAK_ECAPACITY, "dak_global_offload_bytes: overflow %lld B exceeds host capacity %lld B",
                     (long long)over, (long long)host_capacity_bytes);
  *y_req_bytes = over > 0 ? over : 0;
  if (ratio) *ratio = footprint > 0 ? (double)*y_req_bytes / (double)footprint : 0.0;
  return DAK_OK;
}

dak_status dak_decode_ops(const dak_model* m, int32_t batch, int64_t context, int32_t unit_rows, int32_t chunk_tokens,
                          double peak_flops_linear, double peak_flops_attn, dak_op* ops, dak_op_desc* desc,
                          int32_t capacity, int32_t* n_ops) {
  if (!m || !n_ops) return dak::fail(DAK_EINVAL, "dak_decode_ops: NULL argument");
  if (m->family != DAK_MODEL_OPT && m->family != DAK_MODEL_LLAMA) return dak::fail(DAK_EINVAL, "dak_decode_ops: bad family");
  const int tp = m->tp_size > 0 ? m->tp_size : 1;
  if (m->n_layers <= 0 || m->hidden <= 0 || m->n_heads <= 0 || m->n_kv_heads <= 0 || m->head_dim <= 0 || m->ffn <= 0 ||
      m->vocab <= 0 || batch <= 0 || context <= 0 || unit_rows <= 0 || chunk_tokens <= 0)
    return dak::fail(DAK_EINVAL, "dak_decode_ops: sizes must be positive");
  if (!(peak_flops_linear > 0.0) || !(peak_flops_attn > 0.0)) return dak::fail(DAK_EINVAL, "dak_decode_ops: peaks must be positive");
  if (m->n_heads % m->n_kv_heads) return dak::fail(DAK_EINVAL, "dak_decode_ops: n_heads %% n_kv_heads != 0");
  if (m->n_heads % tp || m->n_kv_heads % tp || m->ffn % tp || m->vocab % tp)
    return dak::fail(DAK_EINVAL, "dak_decode_ops: heads / kv heads / ffn / vocab not divisible by tp_size %d", tp);
  const int64_t H = m->hidden, d = m->head_dim;
  const int64_t hq = (int64_t)(m->n_heads / tp) * d, hkv = (int64_t)(m->n_kv_heads / tp) * d;
  const int64_t F = m->ffn / tp, V = m->vocab / tp;

  struct Lin { int32_t role; int64_t M, K; };
  std::vector<Lin> per_layer;
  if (m->fused_qkv) {
    per_layer.push_back({DAK_ROLE_QKV, hq + 2 * hkv, H});
  } else {
    per_layer.push_back({DAK_ROLE_Q, hq, H});
    per_layer.push_back({DAK_ROLE_K, hkv, H});
    per_layer.push_back({DAK_ROLE_V, hkv, H});
  }
  per_layer.push_back({DAK_ROLE_O, H, hq});
  if (m->family == DAK_MODEL_OPT) {
    per_layer.push_back({DAK_ROLE_UP, F, H});    // fc1
    per_layer.push_back({DAK_ROLE_DOWN, H, F});  // fc2
  } else {
    if (m->fused_gate_up) {
      per_layer.push_back({DAK_ROLE_GATE_UP, 2 * F, H});
    } else {
      per_layer.push_back({DAK_ROLE_GATE, F, H});
      per_layer.push_back({DAK_ROLE_UP, F, H});
    }
    per_layer.push_back({DAK_ROLE_DOWN, H, F});
  }
  const int64_t total = (int64_t)m->n_layers * ((int64_t)per_layer.size() + 1) + (m->include_head ? 1 : 0);
  if (total > 0x7fffffff) return dak::fail(DAK_EINVAL, "dak_decode_ops: too many ops");
  *n_ops = (int32_t)total;
  if (!ops && !desc) return DAK_OK;  // count query
  if (capacity < total) return dak::fail(DAK_EINVAL, "dak_decode_ops: capacity %d < %lld ops", capacity, (long long)total);

  const double B = (double)batch;
  int32_t i = 0;
  auto put_linear = [&](int32_t layer, int32_t role, int64_t M, int64_t K) {
    const double flops = 2.0 * B * (double)M * (double)K;  // 2 * tokens * in * out
    if (ops) {
      ops[i].kind = DAK_OP_LINEAR;
      ops[i].reserved = 0;
      ops[i].total_bytes = M * K * 2;         // C_i = weight bytes (P:L422 footnote)
      ops[i].n_units = cdiv(M, unit_rows);    // units of unit_rows output rows (R8)
      ops[i].unit_bytes = (int64_t)unit_rows * K * 2;
      ops[i].t_comp_s = flops / peak_flops_linear;
    }
    if (desc) desc[i] = dak_op_desc{layer, role, M, K, flops};
    ++i;
  };
  const int64_t tok_bytes = 2 * hkv * 2;  // K and V rows of one token, this shard's kv heads
  const int64_t chunks = cdiv(context, chunk_tokens);
  for (int32_t l = 0; l < m->n_layers; ++l) {
    for (const Lin& o : per_layer) put_linear(l, o.role, o.M, o.K);
    // decode attention of the new token over `context` cached tokens per request: C_i = KV bytes
    // (P:L422 footnote), FLOPs 2 (q.K) + 2 (p.V) per token per q head per dim;
    // units = split-KV chunks of chunk_tokens tokens of one request (all this shard's kv heads),
    // mean unit ceil(C / n) (reading R15: every request's last chunk may be short)
    const int64_t C = tok_bytes * (int64_t)batch * context;
    const int64_t n = (int64_t)batch * chunks;
    const double flops = 4.0 * B * (double)context * (double)hq;
    if (ops) {
      ops[i].kind = DAK_OP_ATTENTION;
      ops[i].reserved = 0;
      ops[i].total_bytes = C;
      ops[i].n_units = n;
      ops[i].unit_bytes = cdiv(C, n);
      ops[i].t_comp_s = flops / peak_flops_attn;
    }
    if (desc) desc[i] = dak_op_desc{l, DAK_ROLE_ATTENTION, (int64_t)batch * context, d, flops};
    ++i;
  }
  if (m->include_head) put_linear(-1, DAK_ROLE_HEAD, V, H);
  return DAK_OK;
}

dak_status dak_kv_place(int32_t B, const int32_t* seq_lens, int32_t page_size, int32_t max_pages, int32_t chunk_pages,
                        int64_t host_units, int32_t* block_table, int32_t* n_host_pages, int32_t* n_hbm_pages,
                        int64_t* host_tokens) {
  if (B <= 0 || !seq_lens || page_size <= 0 || max_pages <= 0 || chunk_pages <= 0 || host_units < 0 || !block_table)
    return dak::fail(DAK_EINVAL, "dak_kv_place: bad arguments");
  std::vector<int32_t> filled(B), chunks(B), host_chunks(B, 0);
  int64_t n_chunks = 0;
  int32_t max_ch = 0;
  for (int32_t b = 0; b < B; ++b) {
    if (seq_lens[b] < 0) return dak::fail(DAK_EINVAL, "dak_kv_place: seq_len < 0");
    filled[b] = (int32_t)cdiv(seq_lens[b], page_size);
    if (filled[b] > max_pages) return dak::fail(DAK_EINVAL, "dak_kv_place: request %d needs %d > max_pages pages", b, filled[b]);
    chunks[b] = (int32_t)cdiv(filled[b], chunk_pages);
    n_chunks += chunks[b];
    if (chunks[b] > max_ch) max_ch = chunks[b];
  }
  if (host_units > n_chunks) return dak::fail(DAK_EINVAL, "dak_kv_place: %lld host units > %lld chunks", (long long)host_units, (long long)n_chunks);
  // host units = the oldest chunks, chunk-major: chunk c of requests 0..B-1, then chunk c + 1
  int64_t left = host_units;
  for (int32_t c = 0; c < max_ch && left > 0; ++c)
    for (int32_t b = 0; b < B && left > 0; ++b)
      if (c < chunks[b]) {
        ++host_chunks[b];
        --left;
      }
  int32_t ih = 0, ig = 0;
  int64_t ht = 0;
  for (int32_t b = 0; b < B; ++b) {
    const int64_t hp = std::min<int64_t>((int64_t)host_chunks[b] * chunk_pages, filled[b]);
    for (int32_t p = 0; p < max_pages; ++p)
      block_table[(int64_t)b * max_pages + p] = p < hp ? (int32_t)((uint32_t)ih++ | 0x80000000u) : ig++;
    ht += std::min<int64_t>(hp * page_size, seq_lens[b]);
  }
  if (n_host_pages) *n_host_pages = ih;
  if (n_hbm_pages) *n_hbm_pages = ig;
  if (host_tokens) *host_tokens = ht;
  return DAK_OK;
}

dak_status dak_kv_replace(int32_t B, const int32_t* seq_lens, int32_t page_size, int32_t max_pages, int32_t chunk_pages,
                          int64_t host_units, int32_t host_pool_pages, int32_t hbm_pool_pages, const int32_t* old_table,
                          int32_t* new_table, int32_t* moves, int32_t max_moves, int32_t* n_moves) {
  if (B <= 0 || !seq_lens || page_size <= 0 || max_pages <= 0 || chunk_pages <= 0 || host_units < 0 ||
      host_pool_pages < 0 || hbm_pool_pages < 0 || !old_table || !new_table || max_moves < 0 || (max_moves && !moves) ||
      !n_moves || old_table == new_table)
    return dak::fail(DAK_EINVAL, "dak_kv_replace: bad arguments");
  const int64_t E = (int64_t)B * max_pages;
  // tiers of the fresh chunk-major placement for the new lengths and host units
  std::vector<int32_t> fresh((size_t)E);
  dak_status st = dak_kv_place(B, seq_lens, page_size, max_pages, chunk_pages, host_units, fresh.data(), nullptr, nullptr,
                               nullptr);
  if (st != DAK_OK) return st;
  // free slots: those the old table does not reference, ascending
  std::vector<char> used_h((size_t)host_pool_pages, 0), used_g((size_t)hbm_pool_pages, 0);
  for (int64_t i = 0; i < E; ++i) {
    const uint32_t e = (uint32_t)old_table[i];
    const uint32_t slot = e & 0x7FFFFFFFu;
    if (e & 0x80000000u) {
      if (slot >= (uint32_t)host_pool_pages) return dak::fail(DAK_EINVAL, "dak_kv_replace: old host slot %u >= pool", slot);
      used_h[slot] = 1;
    } else {
      if (slot >= (uint32_t)hbm_pool_pages) return dak::fail(DAK_EINVAL, "dak_kv_replace: old HBM slot %u >= pool", slot);
      used_g[slot] = 1;
    }
  }
  int32_t next_h = 0, next_g = 0, nm = 0;
  for (int64_t i = 0; i < E; ++i) {
    const uint32_t old = (uint32_t)old_table[i];
    const bool want_host = ((uint32_t)fresh[(size_t)i] & 0x80000000u) != 0;
    if (((old & 0x80000000u) != 0) == want_host) {
      new_table[i] = (int32_t)old;
      continue;
    }
    uint32_t ne;
    if (want_host) {
      while (next_h < host_pool_pages && used_h[(size_t)next_h]) ++next_h;
      if (next_h >= host_pool_pages) return dak::fail(DAK_ECAPACITY, "dak_kv_replace: host pool of %d pages is full", host_pool_pages);
      ne = (uint32_t)next_h++ | 0x80000000u;
    } else {
      while (next_g < hbm_pool_pages && used_g[(size_t)next_g]) ++next_g;
      if (next_g >= hbm_pool_pages) return dak::fail(DAK_ECAPACITY, "dak_kv_replace: HBM pool of %d pages is full", hbm_pool_pages);
      ne = (uint32_t)next_g++;
    }
    new_table[i] = (int32_t)ne;
    if (nm >= max_moves) return dak::fail(DAK_EINVAL, "dak_kv_replace: more than max_moves = %d moves", max_moves);
    moves[2 * nm] = (int32_t)old;
    moves[2 * nm + 1] = (int32_t)ne;
    ++nm;
  }
  *n_moves = nm;
  return DAK_OK;
}

dak_status dak_calib_select(const double* table, int32_t n_n_host, int32_t n_window, const int32_t* n_host,
                            const int32_t* window, double tolerance, int32_t* best_i, int32_t* best_j) {
  if (!table || n_n_host <= 0 || n_window <= 0 || !n_host || !window || !best_i || !best_j ||
      !(tolerance >= 0.0 && tolerance < 1.0))
    return dak::fail(DAK_EINVAL, "dak_calib_select: bad arguments");
  const int64_t n = (int64_t)n_n_host * n_window;
  double best = -1.0;
  for (int64_t k = 0; k < n; ++k) best = std::max(best, table[2 * k] + table[2 * k + 1]);
  const double thr = best * (1.0 - tolerance);
  int32_t bi = -1, bj = -1;
  for (int32_t i = 0; i < n_n_host; ++i)
    for (int32_t j = 0; j < n_window; ++j) {
      const int64_t k = (int64_t)i * n_window + j;
      if (table[2 * k] + table[2 * k + 1] < thr) continue;
      if (bi < 0 || n_host[i] < n_host[bi] || (n_host[i] == n_host[bi] && window[j] < window[bj])) {
        bi = i;
        bj = j;
      }
    }
  *best_i = bi;
  *best_j = bj;
  return DAK_OK;
}

}  // extern "C"
