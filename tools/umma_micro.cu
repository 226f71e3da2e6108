// tcgen05.mma issue-rate microbenchmark (development tool): cycles per kind::f16 MMA
// (M = 128, K = 16, SS operands, SWIZZLE_128B K-major) as a function of N, the number of
// independent accumulator chains, and how often tcgen05.commit is issued / waited on.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_micro tools/umma_micro.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(su32(bar)), "r"(ph) : "memory");
}

// mode bit0: commit after every stage (4 MMAs); bit1: wait for that commit before the next stage;
// bit2: A operand from 2 different 16 KB buffers alternating (else the same)
__global__ void __launch_bounds__(128, 1) k(int M, int N, int chains, int stages, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 64);
  unsigned char* A = sm + 1024;              // 2 x [128 rows][128 B]
  unsigned char* B = sm + 1024 + 2 * 16384;  // [256 rows][128 B]
  for (int i = threadIdx.x; i < (2 * 16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      const uint32_t a = su32(A) + ((mode & 4) ? (s & 1) * 16384 : 0), b = su32(B);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma(tmem + (uint32_t)((kk % chains) * N), desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (s | (chains == 1 ? kk : 0)) != 0);
      if (mode & 1) {
        commit(bar);
        if (mode & 2) { wait(bar, ph); ph ^= 1; }
      }
    }
    commit(bar);
    wait(bar, ph);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 1024 + 2 * 16384 + 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 2000;
  printf("grid M N chains mode cycles_per_mma\n");
  for (int grid : {1, 148})
    for (int M : {64, 128})
      for (int N : {8, 64, 128, 256})
        for (int chains : {1, 4})
          for (int mode : {0, 1}) {
            if (chains * N > 512) continue;
            k<<<grid, 128, smem>>>(M, N, chains, stages, mode, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("%d %d %d %d %d %.1f\n", grid, M, N, chains, mode, (double)mx / (stages * 4));
          }
  return 0;
}
