// tcgen05 CTA-pair TS-mode check (development tool): D[256 x N] = A[256 x 64] . B[N x 64]^T with A
// (bf16) in each CTA's TMEM (128 rows per CTA, written by tcgen05.st) and B split by N across the
// pair in shared memory -- the prefill attention's S = Q K^T form on a CTA pair.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma2ts tools/umma2_ts_micro.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool wait_bounded(uint64_t* bar, uint32_t ph) {
  for (long long i = 0; i < (1LL << 26); ++i) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(bar)), "r"(ph) : "memory");
    if (ok) return true;
  }
  return false;
}

__global__ void __launch_bounds__(128, 1) k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int N, int* err) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 64);
  unsigned char* Bs = sm + 1024;  // [N/2 rows][128 B] SW128
  const uint32_t rank = cluster_rank();
  const int nh = N / 2;
  for (int q = threadIdx.x; q < nh * 8; q += blockDim.x) {
    const int r = q >> 3, c = q & 7;
    const uint4 v = reinterpret_cast<const uint4*>(B + (size_t)(nh * rank + r) * 64)[c];
    *reinterpret_cast<uint4*>(Bs + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  // A rows -> TMEM columns 256.. (thread = row of this CTA's 128; bf16 pairs along columns)
  {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = 128 * rank + 32 * w + lane;
    uint32_t v[32];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(A + (size_t)row * 64);
    for (int j = 0; j < 32; ++j) v[j] = src[j];
    const uint32_t ta = tmem + ((uint32_t)(32 * w) << 16) + 256u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + 16u),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t b = su32(Bs);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t bd = desc_sw128(b + kk * 32);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(tmem),
                   "r"(tmem + 256u + 8u * kk), "l"(bd), "r"(idesc), "r"((uint32_t)(kk != 0)));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(bar)),
                 "h"((uint16_t)3) : "memory");
  }
  if (!wait_bounded(bar, 0)) atomicExch(err, 2);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = 128 * rank + 32 * w + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(32 * w) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int e = 0; e < 8; ++e) D[(size_t)row * N + c0 + e] = __uint_as_float(v[e]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

int main() {
  const int Ns[2] = {64, 128};
  for (int ni = 0; ni < 2; ++ni) {
    const int N = Ns[ni];
    __nv_bfloat16 *A, *B;
    float* D;
    int* err;
    cudaMallocManaged(&A, 256 * 64 * 2);
    cudaMallocManaged(&B, N * 64 * 2);
    cudaMallocManaged(&D, 256 * N * 4);
    cudaMallocManaged(&err, 4);
    srand(11 + N);
    for (int i = 0; i < 256 * 64; ++i) A[i] = __float2bfloat16((float)(rand() % 17 - 8));
    for (int i = 0; i < N * 64; ++i) B[i] = __float2bfloat16((float)(rand() % 13 - 6));
    *err = 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 32 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, N, err);
    cudaError_t e2 = cudaDeviceSynchronize();
    if (e != cudaSuccess || e2 != cudaSuccess || *err) {
      printf("N %d: launch %s / sync %s / err %d\n", N, cudaGetErrorString(e), cudaGetErrorString(e2), *err);
      return 1;
    }
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int kk = 0; kk < 64; ++kk) s += (double)__bfloat162float(A[m * 64 + kk]) * __bfloat162float(B[n * 64 + kk]);
        maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
      }
    printf("TS N %d: max |err| %.3g\n", N, maxerr);
  }
  return 0;
}
