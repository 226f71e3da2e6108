"""Pins for the planner oracle (oracle/planner.py) against the paper and the mathematics.

Each test pins the oracle to something other than itself: values printed in the paper
(tests/golden/*.json with citations), closed forms, LP brute force, and the theorem structure.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import planner as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GB = 10**9


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- hardware-level pins

def test_system_peak_gh200():
    g = gold("spec_worked_examples.json")["gh200"]
    assert P.system_peak_bandwidth(g["Bg_gbps"], g["link_gbps"], g["dram_gbps"]) == g["system_peak_gbps"]
    # no remote path -> exactly B_g
    assert P.system_peak_bandwidth(4000, 0, 500) == 4000


def test_machine_balance_h100_example():
    # 989000 GFLOP/s over 4000 GB/s = 247.25 FLOP/B (hand arithmetic)
    assert P.machine_balance(989000e9, 4000e9) == pytest.approx(247.25, rel=1e-15)


# ---------------------------------------------------------------- EB model

def test_eb_examples():
    Bg, Bh = 4000 * GB, 450 * GB
    C = 10 * GB
    assert P.effective_bandwidth(C, 0.0, 0.0, Bg, Bh) == pytest.approx(4000 * GB)
    assert P.effective_bandwidth(C, 0.0, 1.0, Bg, Bh) == pytest.approx(450 * GB)
    # compute-bound B_i = 2000 GB/s, x = 0.5 -> host dominated B_h/x = 900 GB/s
    T = C / (2000 * GB)
    assert P.effective_bandwidth(C, T, 0.5, Bg, Bh) == pytest.approx(900 * GB)


def test_turning_point_is_argmax_on_grid():
    """Acceptance 2: argmax of EB over a 1e-4 grid == B_h/(B_h+B_g) within one step and
    the peak equals B_h + B_g."""
    Bg, Bh = Fraction(4000 * GB), Fraction(450 * GB)
    C = Fraction(10 * GB)
    xs = [Fraction(i, 10000) for i in range(10001)]
    ebs = [P.effective_bandwidth(C, Fraction(0), x, Bg, Bh) for x in xs]
    i = max(range(len(xs)), key=lambda k: ebs[k])
    xstar = Bh / (Bh + Bg)
    assert abs(xs[i] - xstar) <= Fraction(1, 10000)
    assert P.effective_bandwidth(C, Fraction(0), xstar, Bg, Bh) == Bg + Bh  # exact
    assert float(xstar) == pytest.approx(0.1011236, abs=1e-7)


@pytest.mark.parametrize("Bi,xstar", [(2000, 0.225), (450, 1.0)])
def test_compute_bound_threshold(Bi, xstar):
    """x* = min(1, B_h/B_i); pinned as the largest grid x with EB(x) == EB(0)."""
    Bg, Bh = Fraction(4000 * GB), Fraction(450 * GB)
    C = Fraction(10 * GB)
    T = C / (Bi * GB)
    eb0 = P.effective_bandwidth(C, T, Fraction(0), Bg, Bh)
    flat = [Fraction(i, 1000) for i in range(1001) if P.effective_bandwidth(C, T, Fraction(i, 1000), Bg, Bh) == eb0]
    assert float(max(flat)) == pytest.approx(xstar, abs=1e-3)
    assert float(P.turning_point_paper(C, T, Bg, Bh, memory_bound=False)) == pytest.approx(xstar)
    _, a, b = P.thresholds_exact(C, T, Bg, Bh)
    assert a == 0 and float(b / C) == pytest.approx(xstar)


def test_thresholds_reduce_to_paper_on_pure_classes():
    """R1: a_i = b_i = x* C for memory-bound ops; a_i = 0, b_i = C min(1, B_h/B_i) for
    compute-bound ops."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        Bg = Fraction(int(rng.integers(1000, 9000)))
        Bh = Fraction(int(rng.integers(10, 1000)))
        C = Fraction(int(rng.integers(1, 100)))
        # memory-bound: T <= C/(Bg+Bh)
        T = C / (Bg + Bh) * Fraction(int(rng.integers(0, 100)), 100)
        _, a, b = P.thresholds_exact(C, T, Bg, Bh)
        assert a == b == C * Bh / (Bg + Bh)
        # compute-bound: T >= C/Bg
        T = C / Bg * Fraction(int(rng.integers(100, 1000)), 100)
        _, a, b = P.thresholds_exact(C, T, Bg, Bh)
        assert a == 0 and b == C * min(Fraction(1), Bh / (C / T))


# ---------------------------------------------------------------- greedy (App. A)

def _spec_two_ops():
    Bg, Bh = 4000 * GB, 450 * GB
    C = 10 * GB
    # op A memory bound (T ~ 0), op B compute bound with B_i = 2000 GB/s
    return [(C, Fraction(0)), (C, Fraction(C, 2000 * GB))], Bg, Bh


def test_greedy_spec_two_op_examples():
    g = gold("spec_worked_examples.json")["two_op"]
    ops, Bg, Bh = _spec_two_ops()
    for case in g["cases"]:
        Y = Fraction(case["R"]).limit_denominator(1000) * sum(c for c, _ in ops)
        y, phase, obj = P.greedy_exact(ops, Y, Bg, Bh)
        x = [float(y[i] / ops[i][0]) for i in range(2)]
        assert x == pytest.approx(case["x"], abs=1e-6)
        assert float(obj) * 1e3 == pytest.approx(case["objective_ms"], abs=1e-4)


def _random_instance(rng, n_ops):
    Bg = Fraction(int(rng.integers(2000, 8000)))
    Bh = Fraction(int(rng.integers(20, 900)))
    ops = []
    for _ in range(n_ops):
        C = Fraction(int(rng.integers(1, 100)))
        kind = rng.integers(0, 3)
        if kind == 0:  # memory bound
            T = C / (Bg + Bh) * Fraction(int(rng.integers(0, 101)), 100)
        elif kind == 1:  # compute bound
            T = C / Bg * Fraction(int(rng.integers(100, 400)), 100)
        else:  # intermediate band (R1)
            lo, hi = C / (Bg + Bh), C / Bg
            T = lo + (hi - lo) * Fraction(int(rng.integers(1, 100)), 100)
        ops.append((C, T))
    return ops, Bg, Bh


def test_greedy_equals_lp_bruteforce_and_closed_form():
    """Acceptance 3 made exact: on random instances spanning all three regimes, the
    continuous greedy objective equals the exact LP-vertex optimum and the closed form OPT(Y)."""
    rng = np.random.default_rng(2026)
    regimes = [0, 0, 0]
    for trial in range(240):
        ops, Bg, Bh = _random_instance(rng, int(rng.integers(1, 5)))
        Ctot = sum(c for c, _ in ops)
        A = sum(P.thresholds_exact(c, t, Bg, Bh)[1] for c, t in ops)
        Bs = sum(P.thresholds_exact(c, t, Bg, Bh)[2] for c, t in ops)
        reg = trial % 3
        if reg == 0:
            Y = A * Fraction(int(rng.integers(0, 101)), 100)
        elif reg == 1:
            Y = A + (Bs - A) * Fraction(int(rng.integers(0, 101)), 100)
        else:
            Y = Bs + (Ctot - Bs) * Fraction(int(rng.integers(0, 101)), 100)
        regimes[reg] += 1
        _, _, obj = P.greedy_exact(ops, Y, Bg, Bh)
        best, _ = P.brute_force_vertices(ops, Y, Bg, Bh)
        assert obj == best, (ops, Y)
        assert P.closed_form_optimum(ops, Y, Bg, Bh) == best
    assert min(regimes) >= 50


def test_theorem_regime_structure():
    """Theorem 1: in regime 1 every compute-bound op gets x = 0; Theorem 2: in regime 2
    every memory-bound op sits exactly at x* (P:L921); Theorem 3: in regime 3 any feasible plan
    with all x_i >= x_i* has the same objective."""
    rng = np.random.default_rng(7)
    for _ in range(60):
        ops, Bg, Bh = _random_instance(rng, 4)
        th = [P.thresholds_exact(c, t, Bg, Bh) for c, t in ops]
        A = sum(a for _, a, _ in th)
        Bs = sum(b for _, _, b in th)
        Ctot = sum(c for c, _ in ops)
        comp = [i for i, (c, t) in enumerate(ops) if t >= c / Bg]
        mem = [i for i, (c, t) in enumerate(ops) if t <= c / (Bg + Bh)]
        y, _, _ = P.greedy_exact(ops, A / 2, Bg, Bh)
        for i in comp:
            assert y[i] == 0
        y, _, _ = P.greedy_exact(ops, A + (Bs - A) / 2, Bg, Bh)
        for i in mem:
            assert y[i] == th[i][1]
        if Ctot > Bs:
            Y = Bs + (Ctot - Bs) / 3
            _, _, obj = P.greedy_exact(ops, Y, Bg, Bh)
            for _ in range(10):
                w = [Fraction(int(rng.integers(1, 10))) for _ in ops]
                head = [ops[i][0] - th[i][2] for i in range(4)]
                tot = sum(w[i] * head[i] for i in range(4))
                extra = Y - Bs
                yy = [th[i][2] + extra * w[i] * head[i] / tot for i in range(4)]
                o2 = sum(P.op_latency(Fraction(c), Fraction(t), yy[i], Bg, Bh) for i, (c, t) in enumerate(ops))
                assert o2 == obj


def test_greedy_beats_uniform():
    """Acceptance 8 / P:L808: uniform objective >= greedy; equal once R >= sum b_i / sum C_i."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        ops, Bg, Bh = _random_instance(rng, 4)
        Ctot = sum(c for c, _ in ops)
        Bs = sum(P.thresholds_exact(c, t, Bg, Bh)[2] for c, t in ops)
        R = Fraction(int(rng.integers(0, 101)), 100)
        _, g_obj = P.greedy_exact(ops, R * Ctot, Bg, Bh)[1:], P.greedy_exact(ops, R * Ctot, Bg, Bh)[2]
        _, u_obj = P.uniform_allocation(ops, R, Bg, Bh)
        assert u_obj >= g_obj
        # beyond every op's threshold, uniform with x_i >= b_i/C_i is also optimal (Thm 3)
        Rhi = max(Bs / Ctot, max(P.thresholds_exact(c, t, Bg, Bh)[2] / c for c, t in ops))
        _, u2 = P.uniform_allocation(ops, Rhi, Bg, Bh)
        assert u2 == P.greedy_exact(ops, Rhi * Ctot, Bg, Bh)[2]


def test_greedy_boundaries():
    ops, Bg, Bh = _spec_two_ops()
    y, _, _ = P.greedy_exact(ops, 0, Bg, Bh)
    assert all(v == 0 for v in y)
    y, _, _ = P.greedy_exact(ops, sum(c for c, _ in ops), Bg, Bh)
    assert [v for v in y] == [c for c, _ in ops]
    with pytest.raises(ValueError):
        P.greedy_exact(ops, sum(c for c, _ in ops) + 1, Bg, Bh)
    with pytest.raises(ValueError):
        P.greedy_exact([], 0, Bg, Bh)


# ---------------------------------------------------------------- integer-unit greedy (R4-R6)

def _unit_ops(rng, n_ops):
    ops = []
    for _ in range(n_ops):
        n = int(rng.integers(1, 9))
        u = int(rng.integers(1, 40)) * 10**8
        last = int(rng.integers(1, u // 10**8 + 1)) * 10**8
        C = (n - 1) * u + last
        kind = rng.integers(0, 3)
        Bg, Bh = 4000e9, 450e9
        if kind == 0:
            T = 0.0
        elif kind == 1:
            T = C / Bg * float(rng.uniform(1.0, 4.0))
        else:
            T = C / (Bg + Bh) * float(rng.uniform(1.0, 1.12))
        ops.append(dict(n_units=n, unit_bytes=u, total_bytes=C, T=T))
    return ops


def test_units_greedy_properties():
    """EXACT mode: sum host bytes >= Y_req with overshoot < one unit; objective within one unit's
    slope per op of the exact optimum OPT(sum host bytes) (Thm 1-3 + rounding, R4/R5)."""
    rng = np.random.default_rng(5)
    Bg, Bh = 4000e9, 450e9
    for _ in range(300):
        ops = _unit_ops(rng, int(rng.integers(1, 5)))
        Ctot = sum(o["total_bytes"] for o in ops)
        y_req = int(rng.integers(0, Ctot + 1))
        plan = P.plan_units(ops, Bg, Bh, y_req, P.PLAN_EXACT)
        got = sum(plan["host_bytes"])
        assert got >= y_req
        assert got - y_req < max(o["unit_bytes"] for o in ops)
        for i, o in enumerate(ops):
            assert 0 <= plan["host_units"][i] <= o["n_units"]
            assert plan["ratio"][i] == plan["host_units"][i] / o["n_units"]
        exact_ops = [(Fraction(o["total_bytes"]), Fraction(o["T"])) for o in ops]
        opt = P.closed_form_optimum(exact_ops, got, Fraction(Bg), Fraction(Bh))
        slack = sum(Fraction(o["unit_bytes"]) * (1 / Fraction(Bg) + 1 / Fraction(Bh)) for o in ops)
        assert Fraction(plan["objective"]) <= opt + slack + Fraction(1, 10**9)
        assert Fraction(plan["objective"]) >= opt - Fraction(1, 10**9)


def test_units_greedy_vs_integer_bruteforce():
    """Brute force over every integer unit allocation (<=4 ops, <=8 units): the greedy's objective
    is within one unit's slope per op of the best allocation with at least as many host bytes."""
    rng = np.random.default_rng(9)
    Bg, Bh = 4000e9, 450e9
    from itertools import product
    for _ in range(60):
        ops = _unit_ops(rng, int(rng.integers(1, 4)))
        Ctot = sum(o["total_bytes"] for o in ops)
        y_req = int(rng.integers(0, Ctot + 1))
        plan = P.plan_units(ops, Bg, Bh, y_req, P.PLAN_EXACT)
        best = None
        for ks in product(*[range(o["n_units"] + 1) for o in ops]):
            hb = [o["total_bytes"] if k >= o["n_units"] else k * o["unit_bytes"] for k, o in zip(ks, ops)]
            if sum(hb) < y_req:
                continue
            obj = sum(P.op_latency(o["total_bytes"], o["T"], hb[i], Bg, Bh) for i, o in enumerate(ops))
            best = obj if best is None else min(best, obj)
        slack = sum(o["unit_bytes"] * (1 / Bg + 1 / Bh) for o in ops)
        assert plan["objective"] <= best + slack + 1e-12


def test_units_balanced_mode_hits_turning_points():
    """BALANCED mode (north star 'planner's optimal r'): every memory-bound op gets
    round_half_up(x* n) units, x* = B_h/(B_h+B_g)."""
    Bg, Bh = 6555.5e9, 53.0e9
    M, K = 4096, 4096
    op = dict(n_units=M // 8, unit_bytes=8 * K * 2, total_bytes=M * K * 2, T=0.0)
    plan = P.plan_units([op], Bg, Bh, 0, P.PLAN_BALANCED)
    xstar = Fraction(53_000_000_000) / Fraction(6_608_500_000_000)
    expect = math.floor(xstar * (M // 8) + Fraction(1, 2))
    assert plan["host_units"][0] == expect
    assert plan["phase"][0] == 1


def test_units_errors():
    op = dict(n_units=4, unit_bytes=100, total_bytes=400, T=0.0)
    with pytest.raises(P.PlanError) as e:
        P.plan_units([], 1.0, 1.0, 0, 0)
    assert e.value.code == "EINVAL"
    with pytest.raises(P.PlanError) as e:
        P.plan_units([op], 1.0, 1.0, 401, 0)
    assert e.value.code == "ECAPACITY"
    with pytest.raises(P.PlanError) as e:
        P.plan_units([op], 1.0, 1.0, 100, 0, host_capacity=50)
    assert e.value.code == "ECAPACITY"
    with pytest.raises(P.PlanError):
        P.plan_units([dict(op, total_bytes=300)], 1.0, 1.0, 0, 0)  # C not consistent with units


# ---------------------------------------------------------------- capacity -> R (Fig. 8)

def test_fig8_footprint_table():
    """Acceptance 1: KV sizes and global ratios of fig:bw-config."""
    g = gold("fig8_footprint.json")
    kv_tok = P.kv_cache_bytes(48, 56, 128, 1, 1)  # OPT-30B: 48 layers, 7168 = 56 x 128
    assert kv_tok == g["kv_bytes_per_token"]
    for row in g["rows"]:
        kv = P.kv_cache_bytes(48, 56, 128, row["bsz"], row["prompt"] + g["decode_len"])
        assert round(kv / 1e9, 2) == pytest.approx(row["kv_gb"], abs=0.006)
        R = P.global_offload_ratio(g["model_bytes"], kv, g["hbm_bytes"])
        assert float(R) * 100 == pytest.approx(row["ratio_pct"], abs=0.5)


def test_global_ratio_capacity_error():
    with pytest.raises(P.PlanError):
        P.global_offload_ratio(100, 100, 50, host_capacity=10)
    assert P.global_offload_ratio(10, 10, 50) == 0


def test_latency_aware_thresholds_pins():
    """Host latency tau: tau = 0 is the paper's model; for a memory-bound op
    the threshold a = b is the argmin of L(y) = max((C-y)/Bg, y/Bh + tau) (brute force on a
    fine grid, exact Fractions); ops too small to amortise tau (C <= tau Bg) get no host share;
    the double thresholds equal the exact ones to rounding."""
    from fractions import Fraction as Fr
    Bg, Bh = 6700e9, 47e9
    for C, tau in ((102760448, 2.4e-6), (411041792, 2.4e-6), (10_000_000, 2.4e-6), (411041792, 0.0)):
        Ts, a, b = P.thresholds_exact(C, 0, Bg, Bh, tau)
        if C <= tau * Bg:
            assert a == 0
            continue
        assert a == b
        grid = [Fr(C) * k / 20000 for k in range(0, 400)]  # y in [0, 2% of C]
        best = min(grid, key=lambda y: P.op_latency(Fr(C), Fr(0), y, Fr(Bg), Fr(Bh), Fr(tau)))
        assert abs(best - a) <= Fr(C, 20000)
        assert P.op_latency(Fr(C), Fr(0), a, Fr(Bg), Fr(Bh), Fr(tau)) == Ts
        Tsd, ad, bd = P.thresholds_double(float(C), 0.0, Bg, Bh, tau)
        assert abs(ad - float(a)) <= 1e-6 * C and abs(Tsd - float(Ts)) <= 1e-12
    # tau = 0 reproduces R1 bit for bit
    for C, T in ((102760448, 0.0), (411041792, 1e-4), (12345, 3e-9)):
        assert P.thresholds_double(float(C), T, Bg, Bh, 0.0) == P.thresholds_double(float(C), T, Bg, Bh)
