// stream_micro — EXPERIMENT: how fast can a chain of per-op bulk-copy rings stream one op's weights
// at the Llama TP8 b64 shapes? One thread per CTA keeps `stages` copies of `wbytes` (W, HBM,
// rotating > L2) plus an optional `xbytes` copy (x, L2-resident) in flight; the slot is recycled
// as soon as it lands (no consumer). Ops are launched back to back with PDL inside a CUDA graph.
// Prints one JSON line per configuration: GB/s of W bytes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol) : "memory");
}

struct P {
  const char* w;   // this op's weights (contiguous per CTA: [chunks][wbytes])
  const char* x;   // L2-resident operand
  long long per_cta;  // W bytes per CTA
  int wbytes, xbytes, stages, split;  // split: W stage issued as `split` copies
};

__global__ void __launch_bounds__(32, 1) ring(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  unsigned char* ring = sm + 1024;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x != 0) return;
  for (int s = 0; s < p.stages; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint64_t polx;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(polx));
  const long long n = p.per_cta / p.wbytes;
  const char* src = p.w + (long long)blockIdx.x * p.per_cta;
  const int per = p.wbytes + p.xbytes;
  const int pro = (int)(n < p.stages ? n : p.stages);
  const uint32_t part = p.wbytes / p.split;
  for (int i = 0; i < pro; ++i) {
    mbar_expect_tx(&full[i], per);
    for (int j = 0; j < p.split; ++j) bulk(ring + i * per + j * part, src + (long long)i * p.wbytes + j * part, part, &full[i], pol);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.xbytes)
    for (int i = 0; i < pro; ++i) bulk(ring + i * per + p.wbytes, p.x + (i % 64) * p.xbytes, p.xbytes, &full[i], polx);
  int s = 0;
  uint32_t ph = 0;
  for (long long i = pro; i < n + pro; ++i) {
    mbar_wait(&full[s], ph);
    if (i < n) {
      mbar_expect_tx(&full[s], per);
      for (int j = 0; j < p.split; ++j)
        bulk(ring + s * per + j * part, src + i * p.wbytes + j * part, part, &full[s], pol);
      if (p.xbytes) bulk(ring + s * per + p.wbytes, p.x + (i % 64) * p.xbytes, p.xbytes, &full[s], polx);
    }
    if (++s == p.stages) { s = 0; ph ^= 1u; }
  }
}

int main(int argc, char** argv) {
  // usage: stream_micro op_MB grid wKB xKB stages [split] [launches]
  const double op_mb = atof(argv[1]);
  const int grid = atoi(argv[2]), wkb = atoi(argv[3]), xkb = atoi(argv[4]), stages = atoi(argv[5]);
  const int split = argc > 6 ? atoi(argv[6]) : 1;
  const int launches = argc > 7 ? atoi(argv[7]) : 32;
  const int wbytes = wkb * 1024, xbytes = xkb * 1024;
  long long per_cta = (long long)(op_mb * 1e6 / grid) / wbytes * wbytes;
  if (per_cta < wbytes) per_cta = wbytes;
  const long long op_bytes = per_cta * grid;
  const int copies = (int)((4 * 132e6) / op_bytes) + 2;
  std::vector<char*> w(copies);
  for (auto& b : w) CK(cudaMalloc(&b, op_bytes));
  char* x;
  CK(cudaMalloc(&x, 64LL * (xbytes ? xbytes : 16)));
  const int smem = 1024 + stages * (wbytes + xbytes);
  if (smem > 227 * 1024) { printf("{\"error\": \"smem %d\"}\n", smem); return 0; }
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  auto enqueue = [&]() {
    for (int l = 0; l < launches; ++l) {
      P p{w[l % copies], x, per_cta, wbytes, xbytes, stages, split};
      CK(cudaLaunchKernelEx(&cfg, ring, p));
    }
  };
  enqueue();
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  enqueue();
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    CK(cudaEventRecord(e0, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (r && ms < best) best = ms;
  }
  const double us = best * 1e3 / launches;
  printf("{\"op_mb\": %.2f, \"grid\": %d, \"w_kb\": %d, \"x_kb\": %d, \"stages\": %d, \"split\": %d, \"us\": %.2f, \"gbs\": %.0f}\n",
         op_bytes / 1e6, grid, wkb, xkb, stages, split, us, op_bytes / (us * 1e-6) / 1e9);
  return 0;
}
