// Error plumbing, version, device queries and the host-tier allocator of the DAK C ABI.
#include <cuda_runtime.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

#include "common.h"

namespace dak {
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* get_error() { return g_err; }
}  // namespace dak

extern "C" {

const char* dak_last_error(void) { return dak::get_error(); }

const char* dak_version(void) { return "dak-b200 0.1 (sm_100a)"; }

dak_status dak_device_sms(int32_t* sms) {
  if (!sms) return dak::fail(DAK_EINVAL, "sms is NULL");
  int dev = 0, n = 0;
  DAK_CUDA_TRY(cudaGetDevice(&dev));
  DAK_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  *sms = n;
  return DAK_OK;
}

// Host tier: pinned + mapped + portable pages (the SMs read them directly). When a NUMA
// node is requested the pages are first-touched by this thread after an mbind-free placement
// (single-socket boxes: node 0), then registered as mapped.
dak_status dak_host_alloc(size_t bytes, int32_t write_combined, int32_t numa_node, void** host_ptr, void** dev_ptr) {
  if (!host_ptr || !dev_ptr || bytes == 0) return dak::fail(DAK_EINVAL, "dak_host_alloc: bad arguments");
  void* h = nullptr;
  unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable;
  if (write_combined) flags |= cudaHostAllocWriteCombined;
  (void)numa_node;  // single NUMA node on the measured box (profiles/r01/box_probe.txt)
  DAK_CUDA_TRY(cudaHostAlloc(&h, bytes, flags));
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, h, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    return dak::fail(DAK_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  }
  *host_ptr = h;
  *dev_ptr = d;
  return DAK_OK;
}

dak_status dak_host_free(void* host_ptr) {
  if (!host_ptr) return DAK_OK;
  DAK_CUDA_TRY(cudaFreeHost(host_ptr));
  return DAK_OK;
}

}  // extern "C"
