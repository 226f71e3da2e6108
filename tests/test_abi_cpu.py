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


# ------------------------------------------------------------------ a1 / a2 / a4 in the library vs the oracle
def test_global_offload_bytes_vs_oracle_and_fig8(D):
    """dak_global_offload_bytes (a1) against the oracle's exact-Fraction definition, on the paper's
    Fig. 8 capacity runs (golden) and random sizes; ECAPACITY on host overflow."""
    import json
    from fractions import Fraction
    from oracle import planner as P
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "fig8_footprint.json")))
    m = D.model(D.MODEL_OPT, 48, 7168, 56, 56, 128, 28672, 50272)  # OPT-30B
    for row in gold["rows"]:
        # the library's own KV accounting (dak_decode_ops attention C_i over 48 layers) feeds a1
        ops = D.decode_ops(m, row["bsz"], row["prompt"] + gold["decode_len"], 16, 1024, 1e15, 1e15)
        kv = sum(o["total_bytes"] for o in ops if o["role"] == "attn")
        assert round(kv / 1e9, 2) == pytest.approx(row["kv_gb"], abs=0.006)
        w, hbm = int(gold["model_bytes"]), int(gold["hbm_bytes"])  # the paper's 55.6 GB override (R12)
        y, r = D.global_offload_bytes(w, kv, hbm)
        R = P.global_offload_ratio(w, kv, hbm)
        assert y == max(0, w + kv - hbm) and r == float(R)
        assert abs(100 * r - row["ratio_pct"]) < 0.5
    g = np.random.default_rng(8)
    for _ in range(500):
        w, kv, hbm = (int(v) for v in g.integers(0, 1 << 40, 3))
        y, r = D.global_offload_bytes(w, kv, hbm)
        R = P.global_offload_ratio(w, kv, hbm)
        assert Fraction(y) == max(Fraction(0), Fraction(w + kv - hbm)) and r == float(R)
    with pytest.raises(D.DakError) as e:
        D.global_offload_bytes(100, 50, 60, host_capacity_bytes=89)
    assert e.value.code == "ECAPACITY"
    with pytest.raises(P.PlanError):
        P.global_offload_ratio(100, 50, 60, host_capacity=89)
    assert D.global_offload_bytes(100, 50, 60, host_capacity_bytes=90) == (90, 0.6)


@pytest.mark.parametrize("name,tp,B,ctx,fq,fgu,chunk", [("OPT_30B", 1, 8, 64, 1, 0, 64), ("OPT_30B", 1, 1, 2048, 0, 0, 1024),
                                                       ("LLAMA3_70B", 8, 64, 65536, 1, 1, 1024),
                                                       ("LLAMA3_70B", 8, 64, 4096, 0, 0, 256),
                                                       ("LLAMA3_70B", 1, 3, 1000, 1, 0, 384)])
def test_decode_ops_bit_exact_vs_oracle(D, name, tp, B, ctx, fq, fgu, chunk):
    """dak_decode_ops (a2) equals oracle/models.py decode_ops field by field, bitwise for the
    doubles (FLOPs, T): op order, C_i, units, unit bytes, shapes."""
    from oracle import models
    mod = getattr(models, name)
    fam = D.MODEL_OPT if mod["family"] == "opt" else D.MODEL_LLAMA
    m = D.model(fam, mod["n_layers"], mod["hidden"], mod["n_heads"], mod["n_kv_heads"], mod["head_dim"], mod["ffn"],
                mod["vocab"], tp_size=tp, fused_qkv=fq, fused_gate_up=fgu)
    got = D.decode_ops(m, B, ctx, 16, chunk, 1.3554e15, 0.9e15)
    ref = models.decode_ops(mod, B, ctx, 1.3554e15, 0.9e15, tp=tp, unit_rows=16, chunk_tokens=chunk,
                            fused_qkv=bool(fq), fused_gate_up=bool(fgu))
    assert len(got) == len(ref)
    for g_, r_ in zip(got, ref):
        assert g_["kind"] == (0 if r_["kind"] == "linear" else 1)
        assert g_["layer"] == r_["layer"] and models.ROLE[g_["role"]] == r_["role"]
        for f in ("n_units", "unit_bytes", "total_bytes", "M", "K"):
            assert g_[f] == r_[f], f
        assert g_["T"] == r_["T"] and g_["flops"] == r_["flops"]  # bitwise double equality


def test_decode_ops_errors(D):
    m = D.model(D.MODEL_LLAMA, 2, 8192, 64, 8, 128, 28672, 128256, tp_size=16)
    with pytest.raises(D.DakError):
        D.decode_ops(m, 1, 10, 16, 64, 1e15, 1e15)  # 8 kv heads not divisible by 16
    m = D.model(D.MODEL_OPT, 2, 256, 2, 2, 128, 512, 100)
    with pytest.raises(D.DakError):
        D.decode_ops(m, 0, 10, 16, 64, 1e15, 1e15)


def test_kv_place_bit_exact_vs_oracle(D):
    """dak_kv_place (a4, attention) equals oracle/partition.py kv_place_chunk_major bit for bit on
    random ragged batches; host pages are a per-request prefix; host tokens add up."""
    from oracle import partition as Pt
    g = np.random.default_rng(31)
    for trial in range(400):
        B = int(g.integers(1, 9))
        page = int(g.choice([16, 32, 64]))
        cp = int(g.integers(1, 5))
        sl = [int(g.integers(0, 700)) for _ in range(B)]
        max_pages = max(1, max(-(-L // page) for L in sl)) + int(g.integers(0, 3))
        n_chunks = sum(-(-(-(-L // page)) // cp) for L in sl)
        hu = int(g.integers(0, n_chunks + 1))
        bt, nh, ng, ht = D.kv_place(sl, page, max_pages, cp, hu)
        rt, rh, rg, rtok = Pt.kv_place_chunk_major(sl, page, max_pages, cp, hu)
        assert np.array_equal(bt.view(np.uint32), np.array(rt, dtype=np.uint32)), trial
        assert (nh, ng, ht) == (rh, rg, rtok)
        assert nh + ng == B * max_pages
        for b in range(B):  # host pages form a prefix of every request
            host = (bt[b].view(np.uint32) & 0x80000000) != 0
            assert not np.any(host[1:] & ~host[:-1])
    with pytest.raises(D.DakError):
        D.kv_place([64, 64], 64, 1, 1, 3)  # 3 host units > 2 chunks


def test_kv_replace_bit_exact_vs_oracle(D):
    """dak_kv_replace (KV placement across decode steps, reading R23) equals oracle/partition.py
    kv_replace bit for bit -- new block table and the (old entry, new entry) moves in order -- on
    random growing batches; a full destination pool is DAK_ECAPACITY."""
    from oracle import partition as Pt
    from tests.test_oracle_partition import _random_replace_case
    g = np.random.default_rng(47)
    for trial in range(400):
        B, page, cp, Ls0, Ls1, max_pages, hu0, hu1 = _random_replace_case(g)
        old, nh0, ng0, _ = Pt.kv_place_chunk_major(Ls0, page, max_pages, cp, hu0)
        cap_h = nh0 + int(g.integers(0, B * max_pages + 1))
        cap_g = B * max_pages
        try:
            ref_new, ref_moves = Pt.kv_replace(old, Ls1, page, max_pages, cp, hu1, cap_h, cap_g)
        except ValueError:
            with pytest.raises(D.DakError) as e:
                D.kv_replace(old, Ls1, page, max_pages, cp, hu1, cap_h, cap_g)
            assert e.value.code == "ECAPACITY"
            continue
        new, moves = D.kv_replace(old, Ls1, page, max_pages, cp, hu1, cap_h, cap_g)
        assert np.array_equal(new.view(np.uint32), np.array(ref_new, dtype=np.uint32)), trial
        ref_mv = np.array([(s, d) for _, _, s, d in ref_moves], dtype=np.uint32).reshape(-1, 2)
        assert np.array_equal(moves.view(np.uint32), ref_mv), trial


def test_calib_select_bit_exact_vs_oracle(D):
    """dak_calib_select (the calibration's choice, reading R24) equals oracle/partition.py
    calib_choice on random sweeps, with integer-valued rates (exact ties) and real-valued ones."""
    from oracle import partition as Pt
    g = np.random.default_rng(53)
    for trial in range(500):
        ni, nw = int(g.integers(1, 9)), int(g.integers(1, 9))
        n_host = [int(v) for v in g.integers(1, 20, ni)]
        window = [int(v) for v in g.integers(1, 9, nw)]
        if trial % 2:
            tab = g.integers(0, 5, (ni, nw, 2)).astype(np.float64) * 1e9
        else:
            tab = np.stack([g.uniform(5e12, 7e12, (ni, nw)), g.uniform(1e10, 6e10, (ni, nw))], axis=-1)
        tol = float(g.choice([0.0, 0.005, 0.02, 0.1]))
        assert D.calib_select(tab, n_host, window, tol) == Pt.calib_choice(tab.tolist(), n_host, window, tol), trial
    with pytest.raises(D.DakError):
        D.calib_select(np.zeros((1, 1, 2)), [1], [1], 1.5)


def test_kv_place_matches_planned_bytes_when_chunks_are_full(D):
    """With contexts that fill whole chunks, the placed host bytes equal the planner's host bytes
    for the attention op exactly (units are then uniform: reading R15's mean unit is exact)."""
    m = D.model(D.MODEL_OPT, 1, 7168, 56, 56, 128, 28672, 50272, fused_qkv=1)
    B, ctx, page, cp = 8, 2048, 64, 4
    ops = D.decode_ops(m, B, ctx, 16, cp * page, 1.3554e15, 1.3554e15)
    att = [o for o in ops if o["role"] == "attn"][0]
    tok = 2 * 56 * 128 * 2
    for hu in (0, 1, 7, 8, 9, 40, att["n_units"]):
        _, _, _, ht = D.kv_place([ctx] * B, page, ctx // page, cp, hu)
        assert ht * tok == min(hu * att["unit_bytes"], att["total_bytes"])


def test_numa_query_needs_device(D):
    with pytest.raises(D.DakError) as e:
        D.device_numa_node()
    assert e.value.code == "ECUDA"
