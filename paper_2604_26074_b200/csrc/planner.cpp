// dak_plan_ratios — greedy per-op offload planner (PAPER §3.2, App. A).
//
// Integer-unit three-phase water-fill. Compiled with -ffp-contract=off and no fast-math so every
// double operation below is one IEEE rounding in a fixed order (reading R6): the result is
// bit-identical to the oracle's definition (oracle/planner.py:plan_units), which the CPU tests
// check over thousands of random op lists. The oracle is never linked or called from here.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.h"

namespace {

struct OpU {
  int64_t n, u, C;
  double T;
};

inline int64_t unit_bytes_of(int64_t k, const OpU& o) { return k >= o.n ? o.C : k * o.u; }

}  // namespace

extern "C" dak_status dak_plan_ratios(const dak_hw* hw, const dak_op* ops, int32_t n_ops, int64_t y_req,
                                      int32_t mode, dak_op_plan* out, double* objective_s) {
  if (!hw || !ops || !out) return dak::fail(DAK_EINVAL, "dak_plan_ratios: NULL argument");
  if (n_ops <= 0) return dak::fail(DAK_EINVAL, "dak_plan_ratios: ops empty");
  if (mode != DAK_PLAN_EXACT && mode != DAK_PLAN_BALANCED) return dak::fail(DAK_EINVAL, "dak_plan_ratios: bad mode %d", mode);
  const double Bg = hw->hbm_bps;
  // B_h = min(link, host DRAM) (P:L216 footnote)
  const double Bh = hw->link_bps < hw->host_dram_bps ? hw->link_bps : hw->host_dram_bps;
  if (!(Bg > 0.0) || !(Bh > 0.0)) return dak::fail(DAK_EINVAL, "dak_plan_ratios: bandwidths must be positive");
  if (y_req < 0) return dak::fail(DAK_EINVAL, "dak_plan_ratios: y_req < 0");
  const double tau = hw->host_latency_s;
  if (!(tau >= 0.0)) return dak::fail(DAK_EINVAL, "dak_plan_ratios: host_latency_s must be >= 0");

  std::vector<OpU> op(n_ops);
  __int128 total = 0;
  for (int i = 0; i < n_ops; ++i) {
    OpU o{ops[i].n_units, ops[i].unit_bytes, ops[i].total_bytes, ops[i].t_comp_s};
    const __int128 nu = (__int128)o.n * o.u, n1u = (__int128)(o.n - 1) * o.u;
    if (o.n <= 0 || o.u <= 0 || o.C <= 0 || (__int128)o.C > nu || (__int128)o.C <= n1u || !(o.T >= 0.0))
      return dak::fail(DAK_EINVAL, "dak_plan_ratios: op %d has inconsistent units", i);
    op[i] = o;
    total += o.C;
  }
  const int64_t cap = hw->host_capacity_bytes;
  if ((__int128)y_req > total || (cap >= 0 && y_req > cap))
    return dak::fail(DAK_ECAPACITY, "dak_plan_ratios: required host bytes %lld exceed offloadable bytes / host capacity",
                     (long long)y_req);

  // thresholds (reading R1, order R6; host latency tau): T* = max(T, (C + Bh tau)/(Bg+Bh));
  // a = max(0, C - Bg T*); b = max(a, min(C, Bh (T* - tau))). tau = 0 is exactly R1.
  std::vector<int64_t> a_u(n_ops), b_u(n_ops);
  for (int i = 0; i < n_ops; ++i) {
    const double C = (double)op[i].C;
    double Ts = (C + Bh * tau) / (Bg + Bh);
    if (op[i].T > Ts) Ts = op[i].T;
    double a = C - Bg * Ts;
    if (a < 0.0) a = 0.0;
    double b = Bh * (Ts - tau);
    if (b > C) b = C;
    if (b < a) b = a;
    int64_t au = (int64_t)std::floor(a / (double)op[i].u + 0.5);  // round half up
    au = std::min(std::max(au, (int64_t)0), op[i].n);
    int64_t bu = (int64_t)std::floor(b / (double)op[i].u);
    bu = std::min(std::max(bu, au), op[i].n);
    a_u[i] = au;
    b_u[i] = bu;
  }

  int64_t Y = y_req;
  if (mode == DAK_PLAN_BALANCED) {  // offload up to every memory-bound turning point
    int64_t A = 0;
    for (int i = 0; i < n_ops; ++i) A += unit_bytes_of(a_u[i], op[i]);
    if (A > Y) Y = A;
    if (cap >= 0 && Y > cap) Y = std::max(y_req, std::min(Y, cap));
  }

  std::vector<int64_t> units(n_ops, 0), head(n_ops), hb(n_ops), k(n_ops);
  std::vector<int32_t> phase(n_ops, 0);
  std::vector<double> frac(n_ops);
  std::vector<int> order(n_ops);
  int64_t remaining = Y;
  const std::vector<int64_t>* caps[3] = {&a_u, &b_u, nullptr};
  for (int p = 0; p < 3; ++p) {  // phase 1: memory-bound, 2: compute-bound, 3: arbitrary
    if (remaining <= 0) break;
    int64_t H = 0;
    for (int i = 0; i < n_ops; ++i) {
      const int64_t capi = caps[p] ? (*caps[p])[i] : op[i].n;
      head[i] = capi - units[i];
      hb[i] = unit_bytes_of(units[i] + head[i], op[i]) - unit_bytes_of(units[i], op[i]);
      H += hb[i];
    }
    if (H == 0) continue;
    if (remaining >= H) {
      for (int i = 0; i < n_ops; ++i)
        if (head[i] > 0) { units[i] += head[i]; phase[i] = p + 1; }
      remaining -= H;
      continue;
    }
    // proportional to headroom bytes, integer units by largest remainder (reading R5)
    int64_t got = 0;
    for (int i = 0; i < n_ops; ++i) {
      k[i] = 0;
      frac[i] = 0.0;
      if (hb[i] == 0) continue;
      const double share = (double)remaining * (double)hb[i] / (double)H;
      const double q = share / (double)op[i].u;
      int64_t ki = (int64_t)std::floor(q);
      if (ki > head[i]) ki = head[i];
      k[i] = ki;
      frac[i] = q - (double)ki;
    }
    for (int i = 0; i < n_ops; ++i) got += unit_bytes_of(units[i] + k[i], op[i]) - unit_bytes_of(units[i], op[i]);
    for (int i = 0; i < n_ops; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      if (frac[x] != frac[y]) return frac[x] > frac[y];
      return x < y;
    });
    while (got < remaining) {
      bool progressed = false;
      for (int j = 0; j < n_ops; ++j) {
        const int i = order[j];
        if (got >= remaining) break;
        if (k[i] < head[i]) {
          const int64_t before = unit_bytes_of(units[i] + k[i], op[i]);
          k[i] += 1;
          got += unit_bytes_of(units[i] + k[i], op[i]) - before;
          progressed = true;
        }
      }
      if (!progressed) break;
    }
    for (int i = 0; i < n_ops; ++i)
      if (k[i] > 0) { units[i] += k[i]; phase[i] = p + 1; }
    remaining -= got;
  }

  double obj = 0.0;
  for (int i = 0; i < n_ops; ++i) {
    const int64_t hbytes = unit_bytes_of(units[i], op[i]);
    const double hbf = (double)hbytes;
    const double tg = ((double)op[i].C - hbf) / Bg;  // T_g
    const double th = hbf / Bh + (hbytes > 0 ? tau : 0.0);  // T_h (+ host latency)
    double lat = tg > th ? tg : th;
    if (op[i].T > lat) lat = op[i].T;                 // max(T_comp, T_mem)
    out[i].host_units = units[i];
    out[i].host_bytes = hbytes;
    out[i].ratio = (double)units[i] / (double)op[i].n;
    out[i].phase = phase[i];
    out[i].reserved = 0;
    out[i].latency_s = lat;
    obj = obj + lat;
  }
  if (objective_s) *objective_s = obj;
  return DAK_OK;
}
