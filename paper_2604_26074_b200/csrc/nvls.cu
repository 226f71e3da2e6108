// NVLink-SHARP (NVLS) tensor-parallel combine (BASELINE north_star: TP over
// 8 x B200 with the collective over NVLink / NVSwitch).
//
// The row-parallel projections (o, down) of a Megatron layer leave a PARTIAL [rows, cols] output on
// every rank. Instead of ncclAllReduce followed by the residual kernel, the linear writes its partial
// straight into a symmetric NCCL window (ncclMemAlloc + ncclCommWindowRegister: the same offset on
// every rank, bound to an NVSwitch multicast object), and ONE kernel finishes the layer's combine:
//   1. LSA barrier (every rank's partial is written);
//   2. two-shot reduction in the switch: rank r owns rows i with i % world == r and reads their
//      sum with multimem.ld_reduce (fp32 accumulation in the switch, one bf16 rounding), then
//      multimem.st broadcasts it into every rank's copy of the window;
//   3. LSA barrier (every broadcast has landed);
//   4. x += sum (bf16 RNE) and y = RMSNorm(x) * w (the next pre-norm), as dak_allreduce_residual_rmsnorm.
// Each rank's NVLink port moves rows*cols*2 B (its share's reads from the peers plus the broadcast)
// instead of the ring's 2 (world - 1) / world passes; there is no separate collective launch.
//
// The NCCL device API (NCCL >= 2.28: ncclDevCommCreate, symmetric windows, lsaMultimem) is bound at
// run time from the libnccl.so.2 torch loaded; dak_nvls_create returns DAK_EUNSUPPORTED where the
// communicator has no multicast team (one rank, no NVSwitch, NCCL < 2.28) and the caller keeps the
// ncclAllReduce path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>
#include <string.h>

#include "common.h"

namespace dak {
namespace nvls {

struct Api {
  void* h = nullptr;
  ncclResult_t (*mem_alloc)(void**, size_t) = nullptr;
  ncclResult_t (*mem_free)(void*) = nullptr;
  ncclResult_t (*win_register)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*win_deregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclResult_t (*devcomm_create)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*) = nullptr;
  ncclResult_t (*devcomm_destroy)(ncclComm_t, ncclDevComm_t const*) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

static dak_status api(Api** out) {
  static Api a;
  if (!a.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(DAK_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    a.get_version = (decltype(a.get_version))dlsym(h, "ncclGetVersion");
    a.mem_alloc = (decltype(a.mem_alloc))dlsym(h, "ncclMemAlloc");
    a.mem_free = (decltype(a.mem_free))dlsym(h, "ncclMemFree");
    a.win_register = (decltype(a.win_register))dlsym(h, "ncclCommWindowRegister");
    a.win_deregister = (decltype(a.win_deregister))dlsym(h, "ncclCommWindowDeregister");
    a.devcomm_create = (decltype(a.devcomm_create))dlsym(h, "ncclDevCommCreate");
    a.devcomm_destroy = (decltype(a.devcomm_destroy))dlsym(h, "ncclDevCommDestroy");
    a.comm_count = (decltype(a.comm_count))dlsym(h, "ncclCommCount");
    a.comm_user_rank = (decltype(a.comm_user_rank))dlsym(h, "ncclCommUserRank");
    if (!a.get_version || !a.comm_count || !a.comm_user_rank) return fail(DAK_ENCCL, "libnccl.so.2 lacks a required symbol");
    a.h = h;
  }
  int v = 0;
  if (a.get_version(&v) != ncclSuccess || v < 22800 || !a.mem_alloc || !a.win_register || !a.devcomm_create)
    return fail(DAK_EUNSUPPORTED, "NVLS combine needs the NCCL >= 2.28 device API (loaded NCCL %d)", v);
  *out = &a;
  return DAK_OK;
}

struct Handle {
  ncclComm_t comm;
  ncclDevComm dev;
  ncclWindow_t win;
  void* buf;
  size_t bytes;
  int rank, world, n_barriers;
};

constexpr int kThreads = 256;
constexpr int kVec = 8;  // 16-byte chunks per thread (cols <= 256 * 64)

__device__ __forceinline__ uint4 ld_reduce_bf16x8(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_bf16x8(void* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// grid = rows (one CTA per row); the partial [rows, cols] bf16 sits at `offset` in the window
__global__ void __launch_bounds__(kThreads) nvls_residual_rmsnorm_kernel(ncclDevComm dev, ncclWindow_t win, size_t offset,
                                                                         __nv_bfloat16* __restrict__ x, int cols,
                                                                         const __nv_bfloat16* __restrict__ w, float eps,
                                                                         __nv_bfloat16* y) {
  __shared__ float red[kThreads / 32];
  const int r = blockIdx.x;
  const int nc = cols / 8;
  const size_t row_off = offset + (size_t)r * cols * 2;
  {  // 1. every rank has written its partial (kernel boundary + release / acquire at system scope)
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    // 2. two-shot: this rank reduces its rows in the switch and broadcasts the sum
    if (r % dev.lsaSize == dev.lsaRank) {
      char* mc = (char*)ncclGetLsaMultimemPointer(win, row_off, dev);
      for (int c = threadIdx.x; c < nc; c += kThreads) st_bf16x8(mc + (size_t)c * 16, ld_reduce_bf16x8(mc + (size_t)c * 16));
    }
    // 3. every broadcast has landed in every rank's copy
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  // 4. residual + RMSNorm from the local copy (the same arithmetic as residual_rmsnorm_kernel)
  const uint4* pr = reinterpret_cast<const uint4*>((const char*)ncclGetLocalPointer(win, row_off));
  uint4* xr = reinterpret_cast<uint4*>(x) + (size_t)r * nc;
  float f[kVec][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
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
        const float2 q = __bfloat1622float2(oh[j]);
        f[i][2 * j] = q.x;
        f[i][2 * j + 1] = q.y;
        ss += q.x * q.x + q.y * q.y;
      }
      xr[c] = o;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < kThreads / 32; ++i) tot += red[i];  // fixed order
  if (!w) return;  // residual only (no following pre-norm)
  const float rstd = rsqrtf(tot / (float)cols + eps);
  uint4* yr = reinterpret_cast<uint4*>(y) + (size_t)r * nc;
  const uint4* wv = reinterpret_cast<const uint4*>(w);
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    const int c = threadIdx.x + i * kThreads;
    if (c < nc) {
      const uint4 wu = wv[c];
      const __nv_bfloat162* wh = reinterpret_cast<const __nv_bfloat162*>(&wu);
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
}

}  // namespace nvls
}  // namespace dak

using namespace dak;

#define DAK_NCCL_CHECK(expr, what)                                                              \
  do {                                                                                          \
    ncclResult_t r__ = (expr);                                                                  \
    if (r__ != ncclSuccess) return fail(DAK_ENCCL, "%s failed (ncclResult %d)", what, (int)r__); \
  } while (0)

extern "C" {

dak_status dak_nvls_create(void* comm, size_t bytes, int32_t max_rows, void** nvls_out, void** local_buf) {
  if (!comm || !nvls_out || !local_buf || bytes == 0 || max_rows <= 0) return fail(DAK_EINVAL, "dak_nvls_create: bad arguments");
  nvls::Api* a;
  dak_status st = nvls::api(&a);
  if (st != DAK_OK) return st;
  nvls::Handle* h = new nvls::Handle{};
  h->comm = (ncclComm_t)comm;
  h->bytes = (bytes + 4095) / 4096 * 4096;
  h->n_barriers = max_rows;
  DAK_NCCL_CHECK(a->comm_count(h->comm, &h->world), "ncclCommCount");
  DAK_NCCL_CHECK(a->comm_user_rank(h->comm, &h->rank), "ncclCommUserRank");
  if (h->world < 2) {
    delete h;
    return fail(DAK_EUNSUPPORTED, "dak_nvls_create: one rank (no multicast team)");
  }
  // collective calls below: every rank of the communicator makes them in the same order
  DAK_NCCL_CHECK(a->mem_alloc(&h->buf, h->bytes), "ncclMemAlloc");
  DAK_NCCL_CHECK(a->win_register(h->comm, h->buf, h->bytes, &h->win, NCCL_WIN_COLL_SYMMETRIC), "ncclCommWindowRegister");
  ncclDevCommRequirements req;
  memset(&req, 0, sizeof(req));
  req.lsaMultimem = true;
  req.lsaBarrierCount = max_rows;
  DAK_NCCL_CHECK(a->devcomm_create(h->comm, &req, &h->dev), "ncclDevCommCreate");
  if (h->dev.lsaSize != h->world || !h->dev.lsaMultimem.mcBasePtr) {
    a->devcomm_destroy(h->comm, &h->dev);
    a->win_deregister(h->comm, h->win);
    a->mem_free(h->buf);
    delete h;
    return fail(DAK_EUNSUPPORTED, "dak_nvls_create: no NVLink multicast team spanning the communicator");
  }
  *nvls_out = h;
  *local_buf = h->buf;
  return DAK_OK;
}

void* dak_nvls_local(void* nvls) { return nvls ? ((nvls::Handle*)nvls)->buf : nullptr; }

dak_status dak_nvls_destroy(void* nvls) {
  if (!nvls) return DAK_OK;
  nvls::Api* a;
  dak_status st = nvls::api(&a);
  if (st != DAK_OK) return st;
  nvls::Handle* h = (nvls::Handle*)nvls;
  a->devcomm_destroy(h->comm, &h->dev);
  a->win_deregister(h->comm, h->win);
  a->mem_free(h->buf);
  delete h;
  return DAK_OK;
}

dak_status dak_nvls_residual_rmsnorm(void* nvls, size_t offset, void* x, int32_t rows, int32_t cols, const void* norm_w,
                                     float eps, void* y_norm, dak_stream_t stream) {
  nvls::Handle* h = (nvls::Handle*)nvls;
  if (!h || !x || (norm_w && !y_norm) || rows <= 0 || cols <= 0) return fail(DAK_EINVAL, "dak_nvls_residual_rmsnorm: bad arguments");
  if (rows > h->n_barriers) return fail(DAK_EINVAL, "dak_nvls_residual_rmsnorm: rows %d > max_rows %d", rows, h->n_barriers);
  if (cols % 8 || cols > nvls::kThreads * 8 * nvls::kVec || offset % 16 || offset + (size_t)rows * cols * 2 > h->bytes)
    return fail(DAK_EINVAL, "dak_nvls_residual_rmsnorm: cols %% 8, cols <= %d, 16-byte offset inside the window",
                nvls::kThreads * 8 * nvls::kVec);
  if (!aligned16(x) || !aligned16(norm_w) || !aligned16(y_norm)) return fail(DAK_EINVAL, "dak_nvls_residual_rmsnorm: alignment");
  nvls::nvls_residual_rmsnorm_kernel<<<rows, nvls::kThreads, 0, (cudaStream_t)stream>>>(
      h->dev, h->win, offset, (__nv_bfloat16*)x, cols, (const __nv_bfloat16*)norm_w, eps, (__nv_bfloat16*)y_norm);
  DAK_CUDA_TRY(cudaGetLastError());
  return DAK_OK;
}

}  // extern "C"
