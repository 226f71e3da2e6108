// Error plumbing, version, device queries and the host-tier allocator of the DAK C ABI.
#include <cuda_runtime.h>
#include <ctype.h>
#include <errno.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <mutex>
#include <unordered_map>

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

dak_status dak_device_numa_node(int32_t* node) {
  if (!node) return dak::fail(DAK_EINVAL, "node is NULL");
  int dev = 0;
  DAK_CUDA_TRY(cudaGetDevice(&dev));
  char bus[64] = {0};
  DAK_CUDA_TRY(cudaDeviceGetPCIBusId(bus, sizeof(bus), dev));
  for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
  char path[160];
  snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/numa_node", bus);
  int v = -1;
  if (FILE* f = fopen(path, "r")) {
    if (fscanf(f, "%d", &v) != 1) v = -1;
    fclose(f);
  }
  *node = v;
  return DAK_OK;
}

// Host tier: pinned + mapped + portable pages (the SMs read them directly over the link).
// numa_node < 0: cudaHostAlloc (first-touch placement). numa_node >= 0: anonymous pages bound to
// that node with mbind(MPOL_BIND) and faulted in before cudaHostRegister(Mapped | Portable), so a
// GPU reads its host shard from the socket its PCIe link hangs off.
static std::mutex g_reg_mu;
static std::unordered_map<void*, size_t> g_registered;  // mmap'd + registered blocks -> bytes

dak_status dak_host_alloc(size_t bytes, int32_t write_combined, int32_t numa_node, void** host_ptr, void** dev_ptr) {
  if (!host_ptr || !dev_ptr || bytes == 0) return dak::fail(DAK_EINVAL, "dak_host_alloc: bad arguments");
  void* h = nullptr;
  if (numa_node < 0) {
    unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable;
    if (write_combined) flags |= cudaHostAllocWriteCombined;
    DAK_CUDA_TRY(cudaHostAlloc(&h, bytes, flags));
  } else {
    if (write_combined) return dak::fail(DAK_EUNSUPPORTED, "dak_host_alloc: write-combined pages with a NUMA node");
    if (numa_node >= 1024) return dak::fail(DAK_EINVAL, "dak_host_alloc: numa_node %d", numa_node);
    const size_t page = (size_t)sysconf(_SC_PAGESIZE);
    const size_t len = (bytes + page - 1) / page * page;
    h = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h == MAP_FAILED) return dak::fail(DAK_ECUDA, "dak_host_alloc: mmap of %zu B failed (%s)", len, strerror(errno));
    unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
    mask[numa_node / (8 * sizeof(unsigned long))] = 1ul << (numa_node % (8 * sizeof(unsigned long)));
    const long MPOL_BIND_ = 2;
    if (syscall(SYS_mbind, h, len, MPOL_BIND_, mask, (unsigned long)1024, 0u) != 0) {
      const int e = errno;
      munmap(h, len);
      return dak::fail(DAK_EINVAL, "dak_host_alloc: mbind to node %d failed (%s)", numa_node, strerror(e));
    }
    memset(h, 0, len);  // fault every page in on the bound node before pinning
    cudaError_t e = cudaHostRegister(h, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      munmap(h, len);
      return dak::fail(DAK_ECUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> g(g_reg_mu);
    g_registered[h] = len;
  }
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, h, 0);
  if (e != cudaSuccess) {
    dak_host_free(h);
    return dak::fail(DAK_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  }
  *host_ptr = h;
  *dev_ptr = d;
  return DAK_OK;
}

dak_status dak_host_free(void* host_ptr) {
  if (!host_ptr) return DAK_OK;
  size_t len = 0;
  {
    std::lock_guard<std::mutex> g(g_reg_mu);
    auto it = g_registered.find(host_ptr);
    if (it != g_registered.end()) {
      len = it->second;
      g_registered.erase(it);
    }
  }
  if (len) {
    DAK_CUDA_TRY(cudaHostUnregister(host_ptr));
    munmap(host_ptr, len);
    return DAK_OK;
  }
  DAK_CUDA_TRY(cudaFreeHost(host_ptr));
  return DAK_OK;
}

}  // extern "C"
