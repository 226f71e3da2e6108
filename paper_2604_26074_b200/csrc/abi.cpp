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

struct TraceMeta {
  int kind, grid;
  long long a, b;
};
static unsigned long long* g_trace = nullptr;
static int g_trace_cap = 0, g_trace_n = 0;
static TraceMeta* g_trace_meta = nullptr;

unsigned long long* trace_slot(int kind, long long a, long long b, int grid) {
  if (!g_trace || g_trace_n >= g_trace_cap) return nullptr;
  g_trace_meta[g_trace_n] = TraceMeta{kind, grid, a, b};
  return g_trace + (size_t)(g_trace_n++) * kTraceCtas * 4;
}
}  // namespace dak

extern "C" {

const char* dak_last_error(void) { return dak::get_error(); }

const char* dak_version(void) { return "dak-b200 0.1 (sm_100a)"; }

dak_status dak_trace_enable(void* dev_buf, int32_t max_launches) {
  delete[] dak::g_trace_meta;
  dak::g_trace_meta = nullptr;
  dak::g_trace = (unsigned long long*)dev_buf;
  dak::g_trace_cap = dev_buf ? max_launches : 0;
  dak::g_trace_n = 0;
  if (dev_buf) dak::g_trace_meta = new dak::TraceMeta[max_launches > 0 ? max_launches : 1];
  return DAK_OK;
}

dak_status dak_trace_launch(int32_t i, int32_t* kind, int64_t* a, int64_t* b, int32_t* grid) {
  if (i < 0 || i >= dak::g_trace_n || !kind || !a || !b || !grid) return dak::fail(DAK_EINVAL, "dak_trace_launch: bad index");
  *kind = dak::g_trace_meta[i].kind;
  *a = dak::g_trace_meta[i].a;
  *b = dak::g_trace_meta[i].b;
  *grid = dak::g_trace_meta[i].grid;
  return DAK_OK;
}

int32_t dak_trace_count(void) { return dak::g_trace_n; }

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
