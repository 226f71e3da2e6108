"""CPU tests of the C-ABI library: it loads, exports every symbol include/dak.h declares, and its
pure host logic (planner, CTA row ownership) is bit-exact against the oracle. No GPU needed."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def D():
    from paper_2604_26074_b200 import build
    build.build()
    from paper_2604_26074_b200 import dak
    return dak


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "dak.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(dak_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol(D):
    names = _declared_symbols()
    assert "dak_linear" in names and "dak_plan_ratios" in names
    for n in names:
        assert hasattr(D.lib, n), n
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", D._LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    assert set(D.EXPORTED) <= set(names)


def test_version_and_error(D):
    assert "sm_100a" in D.version()


# ------------------------------------------------------------------ planner: bit-exact vs oracle
def _rand_ops(g, n):
    ops = []
    for _ in range(n):
        nu = int(g.integers(1, 600))
        u = int(g.integers(1, 1 << 22)) * 16
        last = int(g.integers(1, u + 1))
        C = (nu - 1) * u + last
        kind = int(g.integers(0, 4))
        Bg = 7.38e12
        if kind == 0:
            T = 0.0
        elif kind == 1:
            T = C / Bg * float(g.uniform(1.0, 6.0))
        elif kind == 2:
            T = C / (Bg + 51.5e9) * float(g.uniform(0.0, 1.01))
        else:
            T = C / (Bg + 51.5e9) * float(g.uniform(1.0, 1.008))
        ops.append(dict(kind=int(g.integers(0, 2)), n_units=nu, unit_bytes=u, total_bytes=C, T=T))
    return ops


def test_planner_bit_exact_vs_oracle(D):
    from oracle import planner as P
    g = np.random.default_rng(12345)
    n_cases = 0
    for trial in range(2500):
        ops = _rand_ops(g, int(g.integers(1, 12)))
        Ctot = sum(o["total_bytes"] for o in ops)
        mode = int(g.integers(0, 2))
        y_req = int(g.integers(0, Ctot + 1)) if trial % 5 else int(g.integers(0, max(1, Ctot // 200)))
        Bg = float(g.choice([7.38e12, 6.5555e12, 4.0e12]))
        Bh = float(g.choice([51.5e9, 450e9, 64e9]))
        dram = Bh * float(g.choice([1.0, 2.0]))
        tau = float(g.choice([0.0, 0.0, 2.4e-6, 1e-5]))  # host latency (latency-aware extension)
        ref = P.plan_units(ops, Bg, min(Bh, dram), y_req, mode, tau=tau)
        got, obj = D.plan_ratios(dict(hbm_bps=Bg, link_bps=Bh, host_dram_bps=dram, host_latency_s=tau), ops, y_req,
                                 mode)
        for i in range(len(ops)):
            assert got[i]["host_units"] == ref["host_units"][i]
            assert got[i]["host_bytes"] == ref["host_bytes"][i]
            assert got[i]["ratio"] == ref["ratio"][i]  # bitwise double equality
            assert got[i]["phase"] == ref["phase"][i]
            assert got[i]["latency"] == ref["latency"][i]
        assert obj == ref["objective"]
        n_cases += 1
    assert n_cases == 2500


def test_planner_model_op_lists_bit_exact(D):
    """Full OPT-30B / Llama-3-70B TP8 decode op lists."""
    from oracle import models, planner as P
    hw = dict(hbm_bps=6555.5e9, link_bps=51.5e9, host_dram_bps=200e9)
    for model, tp, B, ctx in ((models.OPT_30B, 1, 8, 64), (models.LLAMA3_70B, 8, 64, 65536)):
        ops = models.decode_ops(model, B, ctx, 1.3554e15, 1.3554e15, tp=tp)
        Ctot = sum(o["total_bytes"] for o in ops)
        for mode in (0, 1):
            for frac in (0.0, 0.0069, 0.05, 0.4, 1.0):
                y = int(Ctot * frac)
                ref = P.plan_units(ops, hw["hbm_bps"], hw["link_bps"], y, mode)
                got, obj = D.plan_ratios(hw, ops, y, mode)
                assert [g["host_units"] for g in got] == ref["host_units"]
                assert [g["ratio"] for g in got] == ref["ratio"]
                assert obj == ref["objective"]


def test_planner_errors(D):
    hw = dict(hbm_bps=1e12, link_bps=1e10, host_dram_bps=1e10)
    op = dict(n_units=4, unit_bytes=100, total_bytes=400, T=0.0)
    for ops, y, mode, code in (([], 0, 0, "EINVAL"), ([op], 401, 0, "ECAPACITY"), ([op], -1, 0, "EINVAL"),
                                ([dict(op, total_bytes=300)], 0, 0, "EINVAL"), ([op], 0, 7, "EINVAL")):
        with pytest.raises(D.DakError) as e:
            D.plan_ratios(hw, ops, y, mode)
        assert e.value.code == code
    with pytest.raises(D.DakError) as e:
        D.plan_ratios(dict(hw, host_capacity_bytes=50), [op], 100, 0)
    assert e.value.code == "ECAPACITY"
    with pytest.raises(D.DakError) as e:
        D.plan_ratios(dict(hw, hbm_bps=0.0), [op], 0, 0)
    assert e.value.code == "EINVAL"


# ------------------------------------------------------------------ linear launch plan (pure)
@pytest.mark.parametrize("M,h,nh,ng", [(4096, 32, 1, 147), (4096, 0, 0, 148), (7168, 48, 2, 146), (100, 100, 3, 0),
                                       (28672, 208, 1, 147), (50, 7, 2, 5)])
def test_cta_rows_match_oracle(D, M, h, nh, ng):
    from oracle import partition as Pt
    K, kc = 4096, 64
    a = D.linear_args(16 if h else None, 16 if h < M else None, M, K, h, kc, 1, 16, 16,
                      cfg=dict(n_cta_host=nh, n_cta_hbm=ng))
    info = D.linear_query(a)
    assert info["n_cta_host"] == (nh if h else 0) and info["grid"] == info["n_cta_host"] + info["n_cta_hbm"]
    ref = Pt.linear_row_ranges(M, h, info["n_cta_host"], info["n_cta_hbm"])
    got = [D.linear_cta_rows(a, c) for c in range(info["grid"])]
    assert got == ref
    assert info["host_bytes"] == h * K * 2 and info["hbm_bytes"] == (M - h) * K * 2


def test_linear_arg_validation(D):
    bad = [dict(M=0), dict(h=5000), dict(N=4097), dict(K=100), dict(kc=96), dict(kc=8192)]
    for b in bad:
        kw = dict(M=4096, K=4096, h=0, kc=64, N=1)
        kw.update(b)
        a = D.linear_args(16, 16, kw["M"], kw["K"], kw["h"], kw["kc"], kw["N"], 16, 16, cfg=dict(n_cta_hbm=148))
        with pytest.raises(D.DakError) as e:
            D.linear_query(a)
        assert e.value.code in ("EINVAL", "EUNSUPPORTED")
    a = D.linear_args(16, 24, 4096, 4096, 10, 64, 1, 16, 16, cfg=dict(n_cta_hbm=148))  # misaligned hbm pointer
    with pytest.raises(D.DakError):
        D.linear_query(a)


def test_default_kc(D):
    assert D.default_kc(4096, 4096, 147) == 512
    kc = D.default_kc(28672, 7168, 147)
    assert kc == 64 and 7168 % kc == 0
    assert D.default_kc(7168, 28672, 147) == 256
