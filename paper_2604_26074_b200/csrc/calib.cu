// dak_calibrate -- the congestion-control calibration of PAPER §3.3, run online, before
// the decode kernels are launched: "This optimal static window size is calculated via a lightweight
// parameter-sweeping profiler executed prior to kernel launch" and "we perform an offline
// parameter sweep -- fixing the required local GPU SMs while varying the host SMs -- to identify the
// exact SM allocation to the host that maximizes end-to-end throughput".
//
// The probe is the decode kernels' own load path with the compute taken out: one grid of one CTA per
// SM, CTAs [0, n_host) stream the pinned, device-mapped host buffer with `window` bulk copies of
// `chunk` bytes in flight each (the congestion window), the other CTAs stream their slice of the HBM
// buffer with a deep ring (the linear kernels' HBM side). Steady-state runs (every CTA until a
// globaltimer deadline) measure B_g, the saturated link rate and the link latency; each sweep point
// (n_host, window) then times the split GEMV itself (dak_linear, a decode-shaped op of op_mb MiB at
// the balanced ratio r = B_h / (B_g + B_h)) END TO END with n_host host CTAs and n_host x
// window x chunk host bytes in flight, so the op time sees ramp, tail, the host CTAs' own compute
// and congestion alike -- the two curves of P:L510 Fig. 6 folded into one throughput. dak_calib_select (model.cpp) picks the fewest host
// CTAs, then the smallest window, within `tolerance` of the fastest op ("provisions exactly enough
// SMs"). The result feeds the planner (B_g, B_h, tau of dak_hw, measured at the chosen point)
// and the launch configuration (n_cta_host, host_inflight_kb of dak_launch_cfg).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.h"
#include "ptx.cuh"

namespace dak {
namespace cal {

using namespace ptx;

constexpr int kHbmStages = 6;
constexpr int kMaxSlots = 16;
constexpr int kSmem = 227 * 1024;

__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done)
               : "r"(su32(b)), "r"(parity)
               : "memory");
  return done != 0;
}

// stats[cta] = {bytes landed, first issue (ns), last landing (ns), chunks}
// duration_ns > 0: stream until the deadline (steady-state rates); else each CTA streams exactly
// its byte budget (hbm_budget / host_budget bytes) and exits -- one end-to-end split op.
__global__ void __launch_bounds__(32, 1) probe_kernel(const char* hbm, long long hbm_slice, const char* host,
                                                      long long host_bytes, int n_host, int window, int chunk,
                                                      long long duration_ns, long long hbm_budget, long long host_budget,
                                                      long long hbm_off, unsigned long long* stats) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  unsigned char* ring = smem + 1024;
  if (threadIdx.x != 0) return;
  const bool is_host = (int)blockIdx.x < n_host;
  const int slots = is_host ? window : kHbmStages;
  for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const char* base;
  long long span;
  if (is_host) {  // host CTAs start at different offsets of the host buffer
    span = host_bytes / chunk * chunk;
    base = host;
  } else {
    span = hbm_slice / chunk * chunk;
    base = hbm + (long long)(blockIdx.x - n_host) * hbm_slice;
  }
  long long off = is_host ? ((long long)blockIdx.x * 8 * chunk) % span : (hbm_off / chunk * chunk) % span;
  const long long budget_chunks = duration_ns > 0 ? -1 : (is_host ? host_budget : hbm_budget) / chunk;
  if (budget_chunks == 0) {
    if (stats) stats[blockIdx.x * 4 + 0] = 0;
    return;
  }
  auto issue = [&](int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            su32(ring + (size_t)s * chunk)),
        "l"(base + off), "r"(chunk), "r"(su32(&bar[s])), "l"(pol)
        : "memory");
    off += chunk;
    if (off >= span) off = 0;
  };
  const unsigned long long t0 = gtime();
  const unsigned long long deadline = t0 + (unsigned long long)duration_ns;
  long long issued = 0;
  const int first = budget_chunks < 0 || budget_chunks > slots ? slots : (int)budget_chunks;
  for (int s = 0; s < first; ++s) issue(s);
  issued = first;
  unsigned long long bytes = 0, chunks = 0, t_last = t0;
  int s = 0;
  uint32_t ph = 0;
  int in_flight = first;
  bool stop = false;
  while (in_flight > 0) {
    while (!mbar_try(&bar[s], ph)) {
    }
    t_last = gtime();
    bytes += (unsigned long long)chunk;
    ++chunks;
    --in_flight;
    if (!stop && (budget_chunks < 0 ? t_last >= deadline : issued >= budget_chunks)) stop = true;
    if (!stop) {
      issue(s);
      ++issued;
      ++in_flight;
    }
    if (++s == slots) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (stats) {
    stats[blockIdx.x * 4 + 0] = bytes;
    stats[blockIdx.x * 4 + 1] = t0;
    stats[blockIdx.x * 4 + 2] = t_last;
    stats[blockIdx.x * 4 + 3] = chunks;
  }
}

struct Rates {
  double hbm_bps, host_bps, per_chunk_s;
};

// per-tier rate = bytes landed / (last landing - first issue) over the tier's CTAs
static Rates rates(const std::vector<unsigned long long>& st, int grid, int n_host) {
  Rates r{0, 0, 0};
  for (int tier = 0; tier < 2; ++tier) {
    unsigned long long b = 0, lo = ~0ull, hi = 0, ch = 0;
    for (int c = 0; c < grid; ++c) {
      if ((c < n_host) != (tier == 1)) continue;
      b += st[c * 4];
      lo = std::min(lo, st[c * 4 + 1]);
      hi = std::max(hi, st[c * 4 + 2]);
      ch += st[c * 4 + 3];
    }
    const double rate = hi > lo ? (double)b / ((double)(hi - lo) * 1e-9) : 0.0;
    if (tier == 0) r.hbm_bps = rate;
    else {
      r.host_bps = rate;
      r.per_chunk_s = ch ? (double)(hi - lo) * 1e-9 / (double)ch : 0.0;
    }
  }
  return r;
}

}  // namespace cal
}  // namespace dak

using namespace dak;

extern "C" {

dak_status dak_calibrate(const void* hbm_buf, size_t hbm_bytes, const void* host_buf, size_t host_bytes,
                         const dak_calib_opts* opts, dak_calib_result* out, double* table) {
  if (!hbm_buf || !host_buf || !opts || !out || opts->n_n_host <= 0 || opts->n_n_host > 8 || opts->n_window <= 0 ||
      opts->n_window > 8 || opts->chunk_bytes < 1024 || opts->chunk_bytes % 16 || opts->duration_us <= 0 ||
      opts->op_mb < 0 || !aligned16(hbm_buf) || !aligned16(host_buf) || !(opts->tolerance >= 0.0 && opts->tolerance < 1.0))
    return fail(DAK_EINVAL, "dak_calibrate: bad arguments");
  int sms = 0;
  dak_status st = dak_device_sms(&sms);
  if (st != DAK_OK) return st;
  for (int i = 0; i < opts->n_n_host; ++i)
    if (opts->n_host[i] < 1 || opts->n_host[i] >= sms) return fail(DAK_EINVAL, "dak_calibrate: n_host out of range");
  const int chunk = opts->chunk_bytes;
  int max_w = 0;
  for (int j = 0; j < opts->n_window; ++j) {
    if (opts->window[j] < 1 || opts->window[j] > cal::kMaxSlots) return fail(DAK_EINVAL, "dak_calibrate: window out of range");
    max_w = std::max(max_w, opts->window[j]);
  }
  const int smem = 1024 + std::max(cal::kHbmStages, max_w) * chunk;
  if (smem > cal::kSmem) return fail(DAK_EINVAL, "dak_calibrate: window x chunk exceeds shared memory");
  if ((long long)host_bytes < 16LL * chunk) return fail(DAK_EINVAL, "dak_calibrate: host buffer < 16 chunks");
  const long long hbm_slice = (long long)(hbm_bytes / sms) / chunk * chunk;
  if (hbm_slice < (long long)cal::kHbmStages * chunk) return fail(DAK_EINVAL, "dak_calibrate: HBM buffer too small");
  DAK_CUDA_TRY(cudaFuncSetAttribute(cal::probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cal::kSmem));
  cudaStream_t s;
  DAK_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  unsigned long long* d_stats = nullptr;
  if (cudaMalloc(&d_stats, (size_t)sms * 4 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaStreamDestroy(s);
    return fail(DAK_ECUDA, "dak_calibrate: cudaMalloc failed");
  }
  std::vector<unsigned long long> h((size_t)sms * 4);
  const long long dur = (long long)opts->duration_us * 1000;
  const int reps = std::max(1, opts->reps);
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  // steady state: every CTA streams its tier until the deadline (rates of both tiers, concurrently)
  auto steady = [&](int n_host, int window, cal::Rates* r) -> dak_status {
    std::vector<double> hb, lb, pc;
    for (int k = 0; k < reps; ++k) {
      cal::probe_kernel<<<sms, 32, smem, s>>>((const char*)hbm_buf, hbm_slice, (const char*)host_buf,
                                             (long long)host_bytes, n_host, window, chunk, dur, 0, 0, 0, d_stats);
      DAK_CUDA_TRY(cudaGetLastError());
      DAK_CUDA_TRY(cudaMemcpyAsync(h.data(), d_stats, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      DAK_CUDA_TRY(cudaStreamSynchronize(s));
      const cal::Rates q = cal::rates(h, sms, n_host);
      hb.push_back(q.hbm_bps);
      lb.push_back(q.host_bps);
      pc.push_back(q.per_chunk_s);
    }
    *r = {med(hb), med(lb), med(pc)};
    return DAK_OK;
  };
  // end to end: the split GEMV itself (dak_linear, N = 8 decode columns, K = 7168) on a weight of
  // op_mb MiB at the balanced ratio r -- host rows from host_buf, the rest from hbm_buf --
  // with n_host host CTAs and window x chunk host bytes in flight (cfg.host_inflight_kb); timed over
  // a chain of 8 launches. The operands are whatever bytes the buffers hold: only the time is used.
  const long long K = 7168, N = 8;
  const long long op_bytes = (long long)(opts->op_mb > 0 ? opts->op_mb : 384) << 20;
  const long long M = std::max<long long>(256, op_bytes / (2 * K) / 16 * 16);
  const long long y_off = (N * K * 2 + 255) / 256 * 256;       // x [N, K] then y [N, M] at the start of
  const long long xy = (y_off + N * M * 2 + 255) / 256 * 256;  // hbm_buf, the HBM weight rows after them
  auto op = [&](int n_host, int window, double r, double* t_op, long long* hb_bytes, long long* ho_bytes) -> dak_status {
    long long h = (long long)(r * (double)M / 16.0 + 0.5) * 16;
    h = std::max<long long>(16, std::min<long long>(h, M - 16));
    if ((long long)host_bytes < h * K * 2 || (long long)hbm_bytes < xy + (M - h) * K * 2)
      return fail(DAK_EINVAL, "dak_calibrate: buffers too small for the %lld-row probe GEMV", M);
    dak_linear_args la{};
    la.w_host = host_buf;
    la.w_hbm = (const char*)hbm_buf + xy;
    la.M = M;
    la.K = K;
    la.h = h;
    la.N = (int32_t)N;
    la.kc = dak_linear_choose_kc((M - h + sms - n_host - 1) / (sms - n_host), K);
    la.x = hbm_buf;
    la.y = (char*)hbm_buf + y_off;
    la.cfg.n_cta_host = n_host;
    la.cfg.congestion_control = 1;
    la.cfg.pdl = 1;
    la.cfg.host_inflight_kb = (int32_t)((long long)n_host * window * chunk / 1024);
    *hb_bytes = (M - h) * K * 2;
    *ho_bytes = h * K * 2;
    std::vector<double> ts;
    for (int k = 0; k < reps; ++k) {
      DAK_CUDA_TRY(cudaEventRecord(e0, s));
      for (int q = 0; q < 8; ++q) {
        const dak_status st2 = dak_linear(&la, s);
        if (st2 != DAK_OK) return st2;
      }
      DAK_CUDA_TRY(cudaEventRecord(e1, s));
      DAK_CUDA_TRY(cudaEventSynchronize(e1));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1e-3 / 8);
    }
    *t_op = med(ts);
    return DAK_OK;
  };
  dak_status rc = DAK_OK;
  cal::Rates base{}, sat{}, lat{}, fin{};
  std::vector<double> tab((size_t)opts->n_n_host * opts->n_window * 2);
  int bi = 0, bj = 0;
  do {
    if ((rc = steady(0, 1, &base)) != DAK_OK) break;                  // every SM on HBM
    if ((rc = steady(2, max_w, &sat)) != DAK_OK) break;               // the link saturated
    if ((rc = steady(1, 1, &lat)) != DAK_OK) break;                   // one host chunk in flight
    const double r = sat.host_bps / (base.hbm_bps + sat.host_bps);    // balanced ratio
    for (int i = 0; i < opts->n_n_host && rc == DAK_OK; ++i)
      for (int j = 0; j < opts->n_window && rc == DAK_OK; ++j) {
        double t = 0;
        long long hb = 0, ho = 0;
        rc = op(opts->n_host[i], opts->window[j], r, &t, &hb, &ho);
        tab[((size_t)i * opts->n_window + j) * 2 + 0] = t > 0 ? (double)hb / t : 0.0;
        tab[((size_t)i * opts->n_window + j) * 2 + 1] = t > 0 ? (double)ho / t : 0.0;
      }
    if (rc != DAK_OK) break;
    if ((rc = dak_calib_select(tab.data(), opts->n_n_host, opts->n_window, opts->n_host, opts->window, opts->tolerance,
                               &bi, &bj)) != DAK_OK)
      break;
    rc = steady(opts->n_host[bi], opts->window[bj], &fin);            // B_g, B_h at the chosen point
  } while (0);
  cudaFree(d_stats);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  if (rc != DAK_OK) return rc;
  out->n_cta_host = opts->n_host[bi];
  out->window = opts->window[bj];
  out->host_inflight_bytes = (int64_t)out->n_cta_host * out->window * chunk;
  out->hbm_bps = fin.hbm_bps;
  out->link_bps = fin.host_bps;
  out->hbm_alone_bps = base.hbm_bps;
  // one chunk in flight: per-chunk time = latency + the chunk's transfer at the saturated link rate
  out->host_latency_s = std::max(0.0, lat.per_chunk_s - (sat.host_bps > 0 ? (double)chunk / sat.host_bps : 0.0));
  if (table) std::copy(tab.begin(), tab.end(), table);
  return DAK_OK;
}

}  // extern "C"
