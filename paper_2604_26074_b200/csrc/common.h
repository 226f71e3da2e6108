// Internal helpers shared by the DAK C-ABI translation units (not part of the ABI).
#pragma once
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/dak.h"

namespace dak {

// thread-local last-error message (dak_last_error)
void set_error(const char* fmt, ...);
const char* get_error();

inline dak_status fail(dak_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return st;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Launch-timeline tracing (dak_trace_enable): a launch that takes a slot gets a device pointer to
// [kTraceCtas][4] globaltimer stamps; nullptr when tracing is off (the kernels then skip it).
constexpr int kTraceCtas = 1024;
unsigned long long* trace_slot(int kind, long long a, long long b, int grid);
#define DAK_KIND_LINEAR 1
#define DAK_KIND_ATTENTION 2
#define DAK_KIND_COMBINE 3
#define DAK_KIND_APPEND 4
#define DAK_KIND_LAYERNORM 5
#define DAK_KIND_EMBED 6
#define DAK_KIND_REDUCE 7
#define DAK_KIND_PREFILL 8
#define DAK_KIND_RESIDUAL 9
#define DAK_KIND_SILU 10

// dak_linear with the split-K reduce optionally left to the consumer (dak_layer fuses it into the
// next kernel): *ksplit_out = K splits of the launch (1: none, y written); with defer_reduce and
// ksplit > 1 the fp32 partials part[s][n][m] (row stride M) stay in args->workspace.
dak_status linear_enqueue(const dak_linear_args* args, void* stream, bool defer_reduce, int* ksplit_out);
// Llama glue with the split-K reduce of the producing linear fused in (part == nullptr: plain bf16
// input, as the exported dak_rope_kv_append / dak_silu_mul).
dak_status rope_kv_append_part(void* qkv, int64_t row_stride, int32_t B, int32_t Hq, int32_t Hkv, int32_t d,
                               const int32_t* positions, float rope_theta, const int32_t* block_table, int32_t page_size,
                               int32_t max_pages, void* k_hbm, void* v_hbm, void* k_host, void* v_host, int32_t pdl,
                               void* stream, const float* part, int32_t S);
// one rank: x += bf16(sum_s part[s]) (the row-parallel linear's split-K partials, reduced here instead
// of by its reduce kernel), y_norm = RMSNorm(x)
dak_status residual_rmsnorm_part(const float* part, int32_t S, void* x, int32_t rows, int32_t cols, const void* norm_w,
                                 float eps, void* y_norm, int32_t pdl, void* stream);
dak_status silu_mul_part(const void* gu, void* out, int32_t rows, int32_t F, int32_t pdl, void* stream,
                         const float* part, int32_t S);

}  // namespace dak

#define DAK_CUDA_TRY(expr)                                                                       \
  do {                                                                                           \
    cudaError_t e__ = (expr);                                                                    \
    if (e__ != cudaSuccess)                                                                      \
      return ::dak::fail(DAK_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__, __LINE__); \
  } while (0)
