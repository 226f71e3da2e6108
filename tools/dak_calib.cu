// dak_calib — B200 load-path calibration microbenchmarks (component N5).
//
// Decides how SMs read the host tier over the CPU-GPU link (producer
// warp streams tiles into an SMEM ring) and measures the congestion behaviour:
//   1. HBM streaming read: LDG.128 and a cp.async.bulk (TMA engine, UBLKCP) mbarrier ring.
//   2. Host-mapped pinned memory: LDG.128 zero-copy, 1-D cp.async.bulk ring, 2-D TMA tensor
//      (cuTensorMapEncodeTiled on the host pointer) — does each work, at what GB/s, vs #CTAs.
//   3. Concurrent HBM + host CTAs in one grid (host CTAs x window W x chunk): per-tier GB/s.
//   4. Copy-engine H2D for reference.
// Output: one JSON object per line on stdout.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(smem_u32(dst)), "l"(m), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

// ---------------------------------------------------------------- LDG.128 stream
__global__ void ldg_stream(const int4* __restrict__ p, size_t n16, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
    acc.x ^= a.x ^ b.x ^ c.x ^ d.x; acc.y ^= a.y ^ b.y ^ c.y ^ d.y;
    acc.z ^= a.z ^ b.z ^ c.z ^ d.z; acc.w ^= a.w ^ b.w ^ c.w ^ d.w;
  }
  for (; i < n16; i += stride) { int4 a = __ldg(p + i); acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w; }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) sink[0] = 1;
}

// volatile (uncached-style) LDG of host memory, per-CTA contiguous region
__global__ void ldg_region(const int4* __restrict__ p, size_t n16_per_cta, int* sink, uint64_t* t) {
  const int4* q = p + (size_t)blockIdx.x * n16_per_cta;
  uint64_t t0 = gtime();
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = threadIdx.x; i < n16_per_cta; i += 4 * blockDim.x) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; v[u] = j < n16_per_cta ? q[j] : make_int4(0,0,0,0); }
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) sink[0] = 1;
  __syncthreads();
  if (threadIdx.x == 0) { t[2 * blockIdx.x] = t0; t[2 * blockIdx.x + 1] = gtime(); }
}

// ---------------------------------------------------------------- bulk-copy ring (1 producer lane + consumer warps)
// CTAs [0, n_host) read host memory with window `win_host` (<= stages), the rest HBM with all stages.
// Each CTA streams `per_cta` bytes from its own contiguous region in chunks of `chunk` bytes.
struct RingArgs {
  const char* hbm; const char* host; size_t hbm_per_cta; size_t host_per_cta;
  int n_host; int chunk; int stages; int win_host; int use_tma; int tma_rows;
  uint64_t* t; int* sink;
};
__global__ void __launch_bounds__(160) bulk_ring(RingArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 16;
  char* ring = smem + 1024;
  const bool host = (int)blockIdx.x < a.n_host;
  const char* src = host ? a.host + (size_t)blockIdx.x * a.host_per_cta
                         : a.hbm + (size_t)(blockIdx.x - a.n_host) * a.hbm_per_cta;
  const size_t bytes = host ? a.host_per_cta : a.hbm_per_cta;
  const int win = host ? a.win_host : a.stages;
  const int nchunks = (int)(bytes / a.chunk);
  const int n_cons = (blockDim.x / 32) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], n_cons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t t0 = gtime();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nchunks; ++i) {
        int s = i % win; uint32_t ph = (i / win) & 1;
        if (i >= win) mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], a.chunk);
        if (a.use_tma && host) {
          // chunk = tma_rows rows x 128 B, 2-D box over a [rows_total x 64] bf16 view of the region
          int row0 = (int)(((size_t)blockIdx.x * a.host_per_cta + (size_t)i * a.chunk) / 128);
          tma_2d(ring + (size_t)s * a.chunk, &tmap, 0, row0, &full[s]);
        } else {
          bulk_g2s(ring + (size_t)s * a.chunk, src + (size_t)i * a.chunk, a.chunk, &full[s]);
        }
      }
    }
  } else {
    uint32_t acc = 0;
    for (int i = 0; i < nchunks; ++i) {
      int s = i % win; uint32_t ph = (i / win) & 1;
      mbar_wait(&full[s], ph);
      const int4* c = (const int4*)(ring + (size_t)s * a.chunk);
      for (int j = threadIdx.x - 32; j < a.chunk / 16; j += n_cons * 32) { int4 v = c[j]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) a.sink[0] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) { a.t[2 * blockIdx.x] = t0; a.t[2 * blockIdx.x + 1] = gtime(); }
}

// ---------------------------------------------------------------- host helpers
static double span_gbs(const std::vector<uint64_t>& t, int b0, int b1, double bytes) {
  uint64_t lo = UINT64_MAX, hi = 0;
  for (int b = b0; b < b1; ++b) { lo = std::min(lo, t[2 * b]); hi = std::max(hi, t[2 * b + 1]); }
  return hi > lo ? bytes / (double)(hi - lo) : 0.0;  // bytes per ns == GB/s
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  int can_map = 0; CK(cudaDeviceGetAttribute(&can_map, cudaDevAttrCanMapHostMemory, dev));
  int pageable = 0; CK(cudaDeviceGetAttribute(&pageable, cudaDevAttrPageableMemoryAccess, dev));
  printf("{\"test\":\"device\",\"name\":\"%s\",\"sms\":%d,\"l2\":%d,\"smem_optin\":%zu,\"can_map\":%d,\"pageable\":%d,\"pci\":\"%04x:%02x:%02x\"}\n",
         pr.name, pr.multiProcessorCount, l2, pr.sharedMemPerBlockOptin, can_map, pageable, pr.pciDomainID, pr.pciBusID, pr.pciDeviceID);
  fflush(stdout);
  const int SMS = pr.multiProcessorCount;
  int* sink; CK(cudaMalloc(&sink, 64));
  uint64_t* tim; CK(cudaMalloc(&tim, 2 * 1024 * sizeof(uint64_t)));
  std::vector<uint64_t> th(2 * 1024);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));

  const size_t HBM = (size_t)4 << 30;
  char* dbuf; CK(cudaMalloc(&dbuf, HBM)); CK(cudaMemset(dbuf, 1, HBM));
  const size_t HOSTB = (size_t)1 << 30;
  char *hbuf, *hwc;
  CK(cudaHostAlloc(&hbuf, HOSTB, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&hwc, HOSTB, cudaHostAllocMapped | cudaHostAllocPortable | cudaHostAllocWriteCombined));
  memset(hbuf, 3, HOSTB); memset(hwc, 3, HOSTB);
  char *hdev, *hwcdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, hbuf, 0));
  CK(cudaHostGetDevicePointer((void**)&hwcdev, hwc, 0));
  printf("{\"test\":\"uva\",\"host_ptr_eq_dev_ptr\":%d}\n", (int)(hdev == hbuf));

  // 1. HBM LDG stream
  for (int bps : {2, 4, 8}) {
    int grid = SMS * bps;
    ldg_stream<<<grid, 512>>>((const int4*)dbuf, HBM / 16, sink);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) ldg_stream<<<grid, 512>>>((const int4*)dbuf, HBM / 16, sink);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"test\":\"hbm_ldg\",\"ctas\":%d,\"gbs\":%.1f}\n", grid, 5.0 * HBM / (ms * 1e6));
  }
  fflush(stdout);

  // 2. H2D copy engine
  {
    CK(cudaMemcpy(dbuf, hbuf, 256 << 20, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 4; ++r) CK(cudaMemcpyAsync(dbuf, hbuf, 256 << 20, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"test\":\"h2d_copy_engine\",\"bytes\":%d,\"gbs\":%.2f}\n", 256 << 20, 4.0 * (256 << 20) / (ms * 1e6));
  }
  fflush(stdout);

  // 3. host LDG zero-copy vs #CTAs (pinned default and write-combined)
  for (int wc = 0; wc < 2; ++wc) {
    for (int ctas : {1, 2, 4, 8, 16, 32, 64, 148}) {
      size_t per = (size_t)(256 << 20) / ctas / 16;  // 256 MiB total
      const int4* src = (const int4*)(wc ? hwcdev : hdev);
      ldg_region<<<ctas, 512>>>(src, per, sink, tim);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(th.data(), tim, 2 * ctas * sizeof(uint64_t), cudaMemcpyDeviceToHost));
      printf("{\"test\":\"host_ldg\",\"wc\":%d,\"ctas\":%d,\"gbs\":%.2f}\n", wc, ctas, span_gbs(th, 0, ctas, (double)per * 16 * ctas));
      fflush(stdout);
    }
  }

  // 4. bulk ring: HBM only, host only (bulk and TMA), concurrent
  EncodeTiledFn encode = nullptr;
  {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e == cudaSuccess && q == cudaDriverEntryPointSuccess) encode = (EncodeTiledFn)fn;
  }
  CUtensorMap tmap; memset(&tmap, 0, sizeof(tmap));
  int tma_ok = 0;
  if (encode) {
    // view host buffer as [rows, 64] bf16 (128 B rows); box = [64, rows_per_chunk]
    cuuint64_t dims[2] = {64, (cuuint64_t)(HOSTB / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};  // 16 KB box
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)hdev, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    tma_ok = (r == CUDA_SUCCESS);
    printf("{\"test\":\"tma_encode_host\",\"ok\":%d,\"err\":%d}\n", tma_ok, (int)r);
  }
  fflush(stdout);

  auto run_ring = [&](int n_host, int n_hbm, int chunk, int stages, int win, int use_tma, size_t host_per, size_t hbm_per,
                      const char* host_src, const char* tag) {
    RingArgs a;
    a.hbm = dbuf; a.host = host_src; a.hbm_per_cta = hbm_per; a.host_per_cta = host_per;
    a.n_host = n_host; a.chunk = chunk; a.stages = stages; a.win_host = win; a.use_tma = use_tma; a.tma_rows = chunk / 128;
    a.t = tim; a.sink = sink;
    int smem = 1024 + stages * chunk;
    CK(cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = n_host + n_hbm;
    bulk_ring<<<grid, 160, smem>>>(a, tmap);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("{\"test\":\"%s\",\"error\":\"%s\"}\n", tag, cudaGetErrorString(err)); fflush(stdout); exit(2); }
    CK(cudaMemcpy(th.data(), tim, 2 * grid * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    double gh = n_host ? span_gbs(th, 0, n_host, (double)host_per * n_host) : 0.0;
    double gg = n_hbm ? span_gbs(th, n_host, grid, (double)hbm_per * n_hbm) : 0.0;
    printf("{\"test\":\"%s\",\"n_host\":%d,\"n_hbm\":%d,\"chunk\":%d,\"stages\":%d,\"win\":%d,\"tma\":%d,\"host_gbs\":%.2f,\"hbm_gbs\":%.1f}\n",
           tag, n_host, n_hbm, chunk, stages, win, use_tma, gh, gg);
    fflush(stdout);
  };

  // HBM ring alone
  for (int chunk : {16384, 32768}) for (int stages : {4, 6}) {
    if (stages * chunk > 200 * 1024) continue;
    size_t per = (HBM / SMS) / chunk * chunk;
    run_ring(0, SMS, chunk, stages, stages, 0, 0, per, hdev, "hbm_bulk");
  }
  // host ring alone: bulk copies from host-mapped memory
  for (int ctas : {1, 2, 4, 8, 16}) for (int chunk : {4096, 16384, 32768}) for (int win : {1, 2, 4, 6}) {
    size_t per = ((size_t)(128 << 20) / ctas) / chunk * chunk;
    run_ring(ctas, 0, chunk, 6, win, 0, per, 0, hdev, "host_bulk");
  }
  // write-combined
  for (int ctas : {2, 4, 8}) run_ring(ctas, 0, 16384, 6, 4, 0, ((size_t)(128 << 20) / ctas) / 16384 * 16384, 0, hwcdev, "host_bulk_wc");
  // TMA tensor from host
  if (tma_ok) {
    for (int ctas : {1, 2, 4, 8}) for (int win : {2, 4}) {
      size_t per = ((size_t)(128 << 20) / ctas) / 16384 * 16384;
      run_ring(ctas, 0, 16384, 6, win, 1, per, 0, hdev, "host_tma");
    }
  }
  // concurrent: host CTAs + HBM CTAs in one grid (congestion sweep)
  for (int n_host : {1, 2, 4, 8, 16, 32}) for (int win : {1, 2, 4, 6}) {
    int n_hbm = SMS - n_host;
    size_t host_per = ((size_t)(64 << 20) / n_host) / 16384 * 16384;
    size_t hbm_per = ((size_t)(HBM / n_hbm)) / 32768 * 32768;
    // chunk 16 KB for both tiers so the same ring serves either role
    run_ring(n_host, n_hbm, 16384, 6, win, 0, host_per, hbm_per / 16384 * 16384, hdev, "concurrent");
  }
  // concurrent with extra host CTAs co-resident (grid > SMs): 148 HBM + n host
  for (int n_host : {2, 4, 8}) {
    size_t host_per = ((size_t)(64 << 20) / n_host) / 16384 * 16384;
    size_t hbm_per = ((size_t)(HBM / SMS)) / 16384 * 16384;
    run_ring(n_host, SMS, 16384, 6, 4, 0, host_per, hbm_per, hdev, "concurrent_coresident");
  }
  // verify bulk copy content from host (correctness of the path)
  {
    unsigned char* chk; CK(cudaMalloc(&chk, 64));
    CK(cudaFree(chk));
  }
  printf("{\"test\":\"done\"}\n");
  return 0;
}
