// tcgen05 CTA-pair (cta_group::2) micro test (development tool): one cluster of 2 CTAs computes
// D[256 x N] = A[256 x 64] . B[N x 64]^T with ONE M = 256 instruction stream issued by the leader
// CTA; each CTA holds its 128 rows of A and half of B's N rows at the same shared-memory offset.
// Checks the result against the host (which half of B comes from which CTA), then times stages of
// 4 MMAs (K = 64) to get cycles per M = 256 x N x 16 instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma2 tools/umma2_micro.cu
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

// A: [256][64] bf16 row-major; B: [N][64]; D: [256][N] fp32. mode 0: one K = 64 product (check);
// mode 1: `stages` stages of 4 MMAs into the same accumulator, timed (cycles in out[0])
__global__ void __launch_bounds__(128, 1) k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int N, int stages,
                                            long long* out, int* err, int commit_every) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 64);
  unsigned char* As = sm + 1024;          // [128 rows][128 B] SW128
  unsigned char* Bs = sm + 1024 + 16384;  // [N/2 rows][128 B] SW128
  const uint32_t rank = cluster_rank();
  const int nh = N / 2;
  // operands: this CTA's 128 rows of A and rows [nh * rank, nh * rank + nh) of B, 16-byte chunks
  // XOR-swizzled by row & 7 (canonical K-major SWIZZLE_128B)
  for (int q = threadIdx.x; q < 128 * 8; q += blockDim.x) {
    const int r = q >> 3, c = q & 7;
    const uint4 v = reinterpret_cast<const uint4*>(A + (size_t)(128 * rank + r) * 64)[c];
    *reinterpret_cast<uint4*>(As + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  for (int q = threadIdx.x; q < nh * 8; q += blockDim.x) {
    const int r = q >> 3, c = q & 7;
    const uint4 v = reinterpret_cast<const uint4*>(B + (size_t)(nh * rank + r) * 64)[c];
    *reinterpret_cast<uint4*>(Bs + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // both CTAs' operands, barriers and TMEM are ready
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (rank == 0 && threadIdx.x == 0) {
    // kind::f16, D f32, A / B bf16 K-major, N, M = 256
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t a = su32(As), b = su32(Bs);
    const long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = desc_sw128(a + kk * 32), bd = desc_sw128(b + kk * 32);
        const uint32_t acc = (s | kk) != 0;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      if (commit_every)  // a multicast commit per stage to a second barrier (as the GEMM's stage release)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         su32(bar + 1)), "h"((uint16_t)3) : "memory");
    }
    // completion to the barrier at this offset in both CTAs of the pair
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(bar)),
                 "h"((uint16_t)3) : "memory");
    if (!wait_bounded(bar, 0)) atomicExch(err, 1);
    out[0] = clock64() - t0;
  }
  if (!wait_bounded(bar, 0)) atomicExch(err, 2);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads TMEM lanes 32 w .. = this CTA's rows 32 w .. of its 128
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
  const int Ns[3] = {256, 128, 64};
  for (int ni = 0; ni < 3; ++ni) {
    const int N = Ns[ni];
    __nv_bfloat16 *A, *B;
    float* D;
    long long* out;
    int* err;
    cudaMallocManaged(&A, 256 * 64 * 2);
    cudaMallocManaged(&B, N * 64 * 2);
    cudaMallocManaged(&D, 256 * N * 4);
    cudaMallocManaged(&out, 8);
    cudaMallocManaged(&err, 4);
    srand(7 + N);
    for (int i = 0; i < 256 * 64; ++i) A[i] = __float2bfloat16((float)(rand() % 17 - 8));
    for (int i = 0; i < N * 64; ++i) B[i] = __float2bfloat16((float)(rand() % 13 - 6));
    *err = 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 48 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, N, 1, out, err, 0);
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
    cudaLaunchKernelEx(&cfg, k, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, N, 2000, out, err, 0);
    cudaDeviceSynchronize();
    const double c0 = (double)out[0] / 8000.0;
    cudaLaunchKernelEx(&cfg, k, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, N, 2000, out, err, 1);
    cudaDeviceSynchronize();
    printf("N %d: max |err| %.3g; %.1f cycles per M=256 x N x K=16 instruction (2000 stages x 4); %.1f with a multicast commit per stage\n",
           N, maxerr, c0, (double)out[0] / 8000.0);
    cudaFree(A); cudaFree(B); cudaFree(D); cudaFree(out); cudaFree(err);
  }
  return 0;
}
