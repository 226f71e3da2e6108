"""Planner oracle: effective-bandwidth model and the three-phase greedy offload (TEST INFRASTRUCTURE).

Paper passages followed:
  * P:L216 footnote — total system bandwidth = B_g + min(link, host DRAM).
  * EB = C / max(T_comp, T_mem); P:L426 — T_mem = max(T_h, T_g), peak at x* = B_h/(B_h+B_g).
  * compute-bound ops are flat until T_h >= T_comp (threshold x* = min(1, B_h/B_i)).
  * three-phase greedy: (1) memory-bound ops up to their turning point,
    (2) compute-bound ops up to their threshold, (3) arbitrary.
  * Appendix A problem: min sum C_i/EB(x_i) s.t. sum C_i x_i = R sum C_i, 0<=x_i<=1.
  * Theorems 1-3 (regime structure; within-phase split does not matter).

Readings:
  R1  unified thresholds a_i <= b_i (equal to the paper on both pure classes).
  R2  per-op B_i = C_i/T_i.
  R3  Theorem 3's garbled objective read as: beyond b_i every op is host bound.
  R4  integer units: EXACT mode = greedy with sum host bytes >= Y_req.
  R5  within-phase split proportional to headroom, integer units by largest remainder,
      ties to the lower op index.
  R6  fixed IEEE-double formula order (mirrored bit-for-bit by the C++ planner).

Units: bytes and seconds (bandwidths in bytes/s).
"""
from __future__ import annotations

import math
from fractions import Fraction
from itertools import product
from typing import List, Sequence, Tuple

# ----------------------------------------------------------------------------------------------
# hardware-level quantities
# ----------------------------------------------------------------------------------------------


def host_read_bandwidth(link_bw, host_dram_bw):
    """B_h = min(interconnect, host DRAM) — P:L216 footnote."""
    return min(link_bw, host_dram_bw)


def system_peak_bandwidth(hbm_bw, link_bw, host_dram_bw):
    """GPU_HBM_BW + MIN(link, host DRAM) — P:L216 footnote."""
    return hbm_bw + host_read_bandwidth(link_bw, host_dram_bw)


def machine_balance(peak_flops, hbm_bw):
    """FLOP/byte at which an op turns compute bound — P:L382."""
    return peak_flops / hbm_bw


# ----------------------------------------------------------------------------------------------
# per-op effective bandwidth model
# ----------------------------------------------------------------------------------------------


def op_latency(C, T, y, Bg, Bh, tau=0):
    """Latency of an op with C offloadable bytes, compute time T, y bytes on host.

    max(T_comp, T_mem), T_mem = max(T_h, T_g), T_g = (C-y)/B_g, T_h = y/B_h.
    tau (latency-aware extension): a fixed host-path latency paid once the
    op reads any host byte, T_h = y/B_h + tau for y > 0. Works with float or Fraction arguments.
    """
    tg = (C - y) / Bg
    th = y / Bh + (tau if y > 0 else 0)
    return max(T, max(tg, th))


def effective_bandwidth(C, T, x, Bg, Bh):
    """EB(x) = C / max(T_comp, T_mem) with y = x*C on host."""
    return C / op_latency(C, T, x * C, Bg, Bh)


def turning_point_paper(C, T, Bg, Bh, memory_bound: bool):
    """x* as printed in the paper: B_h/(B_h+B_g) for memory-bound ops;
    min(1, B_h/B_i) with B_i = C/T for compute-bound ops (reading R2)."""
    if memory_bound:
        return Bh / (Bh + Bg)
    Bi = C / T
    return min(1, Bh / Bi)


def thresholds_exact(C, T, Bg, Bh, tau=0):
    """Reading R1 (exact arithmetic): T* = max(T, C/(Bg+Bh)), a = max(0, C - Bg T*), b = min(C, Bh T*).

    L(y) decreases with slope -1/Bg on [0,a], is flat (= T*) on [a,b], increases with slope 1/Bh
    on [b, C]. For a memory-bound op (T <= C/(Bg+Bh)) a = b = C*Bh/(Bg+Bh);
    for a compute-bound op (T >= C/Bg) a = 0 and b = C*min(1, Bh/B_i).
    With a host latency tau the balance moves to T* = max(T, (C + Bh tau)/(Bg + Bh)) and the
    host side of the flat segment ends at b = min(C, Bh (T* - tau)) (b >= a); tau = 0 is R1.
    """
    C, T, Bg, Bh, tau = (Fraction(v) for v in (C, T, Bg, Bh, tau))
    Ts = max(T, (C + Bh * tau) / (Bg + Bh))
    a = max(Fraction(0), C - Bg * Ts)
    b = max(a, min(C, Bh * (Ts - tau)))
    return Ts, a, b


def thresholds_double(C: float, T: float, Bg: float, Bh: float, tau: float = 0.0):
    """Reading R6: the same thresholds in IEEE double in this exact operation order
    (the C++ planner mirrors it bit-for-bit; compiled with -ffp-contract=off). tau = 0 gives
    exactly the R1 values (C + 0.0 == C, x - 0.0 == x)."""
    Ts = (C + Bh * tau) / (Bg + Bh)
    if T > Ts:
        Ts = T
    a = C - Bg * Ts
    if a < 0.0:
        a = 0.0
    b = Bh * (Ts - tau)
    if b > C:
        b = C
    if b < a:
        b = a
    return Ts, a, b


# ----------------------------------------------------------------------------------------------
# continuous greedy (exact Fractions) — P:L475-482, Appendix A
# ----------------------------------------------------------------------------------------------


def greedy_exact(ops: Sequence[Tuple], Y, Bg, Bh):
    """Three-phase greedy water-fill in exact arithmetic.

    ops: sequence of (C_i bytes, T_i seconds). Y: total host bytes (= R * sum C_i).
    Phase 1 fills the decreasing segments [0, a_i] (memory-bound turning points),
    phase 2 the flat segments [a_i, b_i] (compute-bound thresholds), phase 3 the rest
    (P:L481). Within a phase the budget is split proportionally to segment headroom (R5).
    Returns (y list of Fractions, phase list, objective Fraction).
    """
    Bg, Bh, Y = Fraction(Bg), Fraction(Bh), Fraction(Y)
    Cs = [Fraction(c) for c, _ in ops]
    if not ops:
        raise ValueError("ops empty")
    if Y < 0 or Y > sum(Cs):
        raise ValueError("Y outside [0, sum C]")  # S:L215 (R > 1)
    th = [thresholds_exact(c, t, Bg, Bh) for c, t in ops]
    seg_hi = [[a for _, a, _ in th], [b for _, _, b in th], Cs]
    y = [Fraction(0)] * len(ops)
    phase = [0] * len(ops)
    rem = Y
    for p in range(3):
        head = [seg_hi[p][i] - y[i] for i in range(len(ops))]
        H = sum(head)
        if H == 0 or rem == 0:
            continue
        take = min(rem, H)
        for i in range(len(ops)):
            if head[i] > 0:
                y[i] += take * head[i] / H
                phase[i] = p + 1
        rem -= take
    obj = sum(op_latency(Fraction(c), Fraction(t), y[i], Bg, Bh) for i, (c, t) in enumerate(ops))
    return y, phase, obj


def closed_form_optimum(ops: Sequence[Tuple], Y, Bg, Bh):
    """OPT(Y) = sum_i max(T_i, C_i/Bg) - min(Y, A)/Bg + max(0, Y - B)/Bh, A = sum a_i, B = sum b_i.

    Follows from Theorems 1-3: Y spent below A lowers the total at slope 1/Bg
    (Thm 1), between A and B costs nothing (Thm 2), beyond B costs 1/Bh per byte (Thm 3, R3).
    """
    Bg, Bh, Y = Fraction(Bg), Fraction(Bh), Fraction(Y)
    base = Fraction(0)
    A = Fraction(0)
    Bsum = Fraction(0)
    for c, t in ops:
        c, t = Fraction(c), Fraction(t)
        base += max(t, c / Bg)
        _, a, b = thresholds_exact(c, t, Bg, Bh)
        A += a
        Bsum += b
    return base - min(Y, A) / Bg + max(Fraction(0), Y - Bsum) / Bh


def brute_force_vertices(ops: Sequence[Tuple], Y, Bg, Bh):
    """Exact optimum of the Appendix-A problem by LP-vertex enumeration.

    Each L_i is convex piecewise linear (a max of affine pieces), so some optimum has every op
    but one at a breakpoint of its own L_i. Candidate breakpoints are taken straight from the
    pieces (0, C, C - Bg T, C Bh/(Bg+Bh), Bh T, clipped to [0, C]) — independent of the
    threshold formulas used by the greedy. Returns (objective, y tuple).
    """
    Bg, Bh, Y = Fraction(Bg), Fraction(Bh), Fraction(Y)
    cand = []
    for c, t in ops:
        c, t = Fraction(c), Fraction(t)
        pts = {Fraction(0), c, c - Bg * t, c * Bh / (Bg + Bh), Bh * t}
        cand.append(sorted(p for p in pts if 0 <= p <= c))
    n = len(ops)
    best = None
    for j in range(n):
        others = [cand[i] for i in range(n) if i != j]
        for choice in product(*others):
            rest = Y - sum(choice)
            cj = Fraction(ops[j][0])
            if rest < 0 or rest > cj:
                continue
            y = list(choice)
            y.insert(j, rest)
            obj = sum(op_latency(Fraction(c), Fraction(t), y[i], Bg, Bh) for i, (c, t) in enumerate(ops))
            if best is None or obj < best[0]:
                best = (obj, tuple(y))
    return best


def uniform_allocation(ops: Sequence[Tuple], R, Bg, Bh):
    """Uniform baseline: every x_i = R. Returns (y list, objective)."""
    R = Fraction(R)
    y = [Fraction(c) * R for c, _ in ops]
    obj = sum(op_latency(Fraction(c), Fraction(t), y[i], Fraction(Bg), Fraction(Bh)) for i, (c, t) in enumerate(ops))
    return y, obj


# ----------------------------------------------------------------------------------------------
# integer-unit greedy in IEEE double — the definition the C ABI's dak_plan_ratios must match
# bit-for-bit (readings R4, R5, R6)
# ----------------------------------------------------------------------------------------------

PLAN_EXACT = 0
PLAN_BALANCED = 1


class PlanError(ValueError):
    def __init__(self, code: str, msg: str):
        super().__init__(msg)
        self.code = code  # "EINVAL" | "ECAPACITY"


def _unit_bytes_of(k: int, n: int, u: int, C: int) -> int:
    """Host bytes of the leading k units (tile row 0 is the host row; R7)."""
    return C if k >= n else k * u


def plan_units(ops: Sequence[dict], Bg: float, Bh: float, y_req: int, mode: int,
               host_capacity: int | None = None, tau: float = 0.0):
    """Greedy per-op offload plan at unit granularity (P:L475-482 with readings R4-R6).

    ops: dicts with n_units, unit_bytes, total_bytes (ints) and T (seconds, float).
    Returns dict(host_units, host_bytes, ratio, phase, latency, objective).

    Steps:
      1. thresholds (R6 double order); a_u = clamp(floor(a/u + 0.5), 0, n) (round half up,
         S:L323), b_u = clamp(floor(b/u), a_u, n).
      2. Y = y_req (EXACT) or max(y_req, sum bytes(a_u)) (BALANCED: offload up to the
         memory-bound balance points).
      3. phases 1..3 with headrooms a_u, b_u - a_u, n - b_u: a phase whose headroom bytes fit
         in the remaining budget is taken whole; otherwise the remaining budget is split
         proportionally to headroom bytes: k_i = floor(share_i/u_i) then +1 unit in descending
         fractional remainder (ties: lower index) until sum bytes >= remaining (R5).
    """
    if not ops:
        raise PlanError("EINVAL", "ops empty")
    if not (Bg > 0.0 and Bh > 0.0):
        raise PlanError("EINVAL", "bandwidths must be positive")
    if mode not in (PLAN_EXACT, PLAN_BALANCED):
        raise PlanError("EINVAL", "bad mode")
    if y_req < 0:
        raise PlanError("EINVAL", "y_req < 0")
    n_ops = len(ops)
    n = [int(o["n_units"]) for o in ops]
    u = [int(o["unit_bytes"]) for o in ops]
    C = [int(o["total_bytes"]) for o in ops]
    T = [float(o["T"]) for o in ops]
    for i in range(n_ops):
        if n[i] <= 0 or u[i] <= 0 or C[i] <= 0 or C[i] > n[i] * u[i] or C[i] <= (n[i] - 1) * u[i] or T[i] < 0.0:
            raise PlanError("EINVAL", f"op {i}: bad units")
    total = sum(C)
    if y_req > total or (host_capacity is not None and y_req > host_capacity):
        raise PlanError("ECAPACITY", "required host bytes exceed offloadable bytes / host capacity")

    a_u, b_u = [], []
    for i in range(n_ops):
        _, a, b = thresholds_double(float(C[i]), T[i], Bg, Bh, tau)
        au = math.floor(a / float(u[i]) + 0.5)
        au = min(max(au, 0), n[i])
        bu = math.floor(b / float(u[i]))
        bu = min(max(bu, au), n[i])
        a_u.append(int(au))
        b_u.append(int(bu))

    Y = int(y_req)
    if mode == PLAN_BALANCED:
        A_bytes = sum(_unit_bytes_of(a_u[i], n[i], u[i], C[i]) for i in range(n_ops))
        if A_bytes > Y:
            Y = A_bytes
        if host_capacity is not None and Y > host_capacity:
            Y = max(int(y_req), min(Y, host_capacity))

    units = [0] * n_ops
    phase = [0] * n_ops
    remaining = Y
    caps = [a_u, b_u, n]
    for p in range(3):
        if remaining <= 0:
            break
        head = [caps[p][i] - units[i] for i in range(n_ops)]
        hb = [_unit_bytes_of(units[i] + head[i], n[i], u[i], C[i]) - _unit_bytes_of(units[i], n[i], u[i], C[i])
              for i in range(n_ops)]
        H = sum(hb)
        if H == 0:
            continue
        if remaining >= H:
            for i in range(n_ops):
                if head[i] > 0:
                    units[i] += head[i]
                    phase[i] = p + 1
            remaining -= H
            continue
        # proportional split with largest remainder
        k = [0] * n_ops
        frac = [0.0] * n_ops
        for i in range(n_ops):
            if hb[i] == 0:
                continue
            share = float(remaining) * float(hb[i]) / float(H)
            q = share / float(u[i])
            ki = math.floor(q)
            if ki > head[i]:
                ki = head[i]
            k[i] = int(ki)
            frac[i] = q - float(ki)
        got = sum(_unit_bytes_of(units[i] + k[i], n[i], u[i], C[i]) - _unit_bytes_of(units[i], n[i], u[i], C[i])
                  for i in range(n_ops))
        order = sorted(range(n_ops), key=lambda i: (-frac[i], i))
        while got < remaining:
            progressed = False
            for i in order:
                if got >= remaining:
                    break
                if k[i] < head[i]:
                    before = _unit_bytes_of(units[i] + k[i], n[i], u[i], C[i])
                    k[i] += 1
                    got += _unit_bytes_of(units[i] + k[i], n[i], u[i], C[i]) - before
                    progressed = True
            if not progressed:
                break
        for i in range(n_ops):
            if k[i] > 0:
                units[i] += k[i]
                phase[i] = p + 1
        remaining -= got

    host_bytes = [_unit_bytes_of(units[i], n[i], u[i], C[i]) for i in range(n_ops)]
    ratio = [float(units[i]) / float(n[i]) for i in range(n_ops)]
    latency = []
    obj = 0.0
    for i in range(n_ops):
        hbf = float(host_bytes[i])
        tg = (float(C[i]) - hbf) / Bg
        th = hbf / Bh + (tau if host_bytes[i] > 0 else 0.0)
        lat = tg if tg > th else th
        if T[i] > lat:
            lat = T[i]
        latency.append(lat)
        obj = obj + lat
    return dict(host_units=units, host_bytes=host_bytes, ratio=ratio, phase=phase,
                latency=latency, objective=obj, y_target=Y, a_units=a_u, b_units=b_u)


# ----------------------------------------------------------------------------------------------
# capacity -> global offload ratio
# ----------------------------------------------------------------------------------------------


def kv_cache_bytes(n_layers, n_kv_heads, head_dim, batch, seq_tokens, dtype_bytes=2):
    """2 (K and V) x layers x kv heads x head_dim x batch x tokens x dtype."""
    return 2 * n_layers * n_kv_heads * head_dim * batch * seq_tokens * dtype_bytes


def global_offload_ratio(weight_bytes, kv_bytes, hbm_capacity, host_capacity=None):
    """R = clamp((footprint - HBM)/footprint, 0, 1); error if overflow > host capacity."""
    footprint = Fraction(weight_bytes) + Fraction(kv_bytes)
    over = footprint - Fraction(hbm_capacity)
    if host_capacity is not None and over > host_capacity:
        raise PlanError("ECAPACITY", "overflow exceeds host capacity")
    if over <= 0:
        return Fraction(0)
    return min(Fraction(1), over / footprint)
