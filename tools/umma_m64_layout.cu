// Probe (development tool): where does a tcgen05.mma.cta_group::1.kind::f16 with M = 64 put row m of
// D in TMEM? A[m][0] = m + 1, A[m][1] = 256; B[n][0] = 1, B[n][1] = n + 1 -> D[m][n] = m + 1 + 256 (n + 1).
// Each of the 4 warps reads TMEM lanes 32w .. 32w + 31, columns 0..7 (tcgen05.ld.32x32b.x8) and the
// host prints, per lane, the decoded (m, n) of column 0..7 (or "-" for untouched lanes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/m64 tools/umma_m64_layout.cu
#include <cuda_bf16.h>
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

__global__ void k(int M, float* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 64);
  unsigned char* A = sm + 1024;          // [128 rows][128 B], SW128 K-major
  unsigned char* B = sm + 1024 + 16384;  // [8 rows][128 B]
  for (int i = threadIdx.x; i < (16384 + 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0u;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int m = threadIdx.x;  // chunk 0 of row m sits at (0 ^ (m & 7)) << 4
    __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(A + (m >> 3) * 1024 + (m & 7) * 128 + ((0 ^ (m & 7)) << 4));
    row[0] = __float2bfloat16((float)(m + 1));
    row[1] = __float2bfloat16(256.f);
  }
  if (threadIdx.x < 8) {
    const int n = threadIdx.x;
    __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(B + (n & 7) * 128 + ((0 ^ (n & 7)) << 4));
    row[0] = __float2bfloat16(1.f);
    row[1] = __float2bfloat16((float)(n + 1));
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(8 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                 "l"(desc_sw128(su32(A))), "l"(desc_sw128(su32(B))), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
    asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W; }" ::"r"(su32(bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 8; ++c) out[(32 * w + lane) * 8 + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * 4);
  const int smem = 1024 + 16384 + 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int M : {128, 64}) {
    cudaMemset(d, 0, 128 * 8 * 4);
    k<<<1, 128, smem>>>(M, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float h[128 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M = %d: lane: (m,n) of columns 0..7\n", M);
    for (int l = 0; l < 128; ++l) {
      printf("%3d:", l);
      for (int c = 0; c < 8; ++c) {
        const float f = h[l * 8 + c];
        if (f == 0.f) { printf("   -   "); continue; }
        const int n1 = (int)(f / 256.f);
        const int m1 = (int)(f - 256.f * n1);
        printf(" (%2d,%d)", m1 - 1, n1 - 1);
      }
      printf("\n");
    }
  }
  return 0;
}
