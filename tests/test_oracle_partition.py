"""Pins for oracle/partition.py: SPEC worked examples, Table 1 (paper-printed), invariants."""
import json
import os

import pytest

from oracle import partition as Pt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_partition_examples():
    for ex in gold("spec_worked_examples.json")["partition"]:
        if ex.get("error"):
            with pytest.raises(ValueError):
                Pt.partition_op(ex["M"], ex["tile_m"], ex["x"])
            continue
        assert Pt.partition_op(ex["M"], ex["tile_m"], ex["x"]) == (ex["host"], ex["gpu"])


def test_partition_conservation_and_accuracy():
    """Tile conservation and |host/rows - x| <= 1/rows."""
    from fractions import Fraction
    for M in (128, 1000, 4096, 7168, 28672):
        for tm in (8, 16, 128):
            rows = -(-M // tm)
            for k in range(0, 101, 7):
                x = Fraction(k, 100)
                h, g = Pt.partition_op(M, tm, x)
                assert h + g == rows
                assert abs(Fraction(h, rows) - x) <= Fraction(1, rows)


def test_wave_alignment_example():
    ex = gold("spec_worked_examples.json")["wave_alignment"]
    assert Pt.wave_aligned_sms(ex["host_rows"], ex["share"]) == ex["n_sm_host"]
    # brute force over the reading R9: largest even divisor that keeps the wave count
    for rows in range(1, 60):
        for share in range(1, 20):
            n = Pt.wave_aligned_sms(rows, share)
            waves = -(-rows // share)
            ok = [d for d in range(1, share + 1) if rows % d == 0 and -(-rows // d) == waves]
            assert n == (max(ok) if ok else share)
            # alignment never increases the number of waves
            assert -(-rows // n) == waves


def test_assign_sms_cap_and_zero():
    assert Pt.assign_sms(0, 100, 132) == (0, 132)
    n_host, n_gpu = Pt.assign_sms(20, 30, 132, cap=8)  # cap from P:L524 congestion onset
    assert n_host <= 8 and n_host + n_gpu == 132
    with pytest.raises(ValueError):
        Pt.assign_sms(1, 1, 1)


def test_cluster_fetch_counts():
    for ex in gold("spec_worked_examples.json")["clusters"]:
        assert Pt.fetches_per_row(ex["consumers"], ex["multicast"], ex["cluster_max"]) == ex["fetches"]


def test_table1_read_amplification():
    """Table 1 reproduced exactly: traffic = ceil(N/256) x 7168^2 x 2 B, printed in
    decimal MB / GB; the true amplification is N/256 (the '98 MB' matrix is 98 MiB)."""
    g = gold("table1_read_amplification.json")
    host_bytes = g["M"] * g["K"] * g["dtype_bytes"]
    assert host_bytes == 98 * 2**20
    prev = None
    for row in g["rows"]:
        t = Pt.host_traffic(host_bytes, row["N"], g["tile_n"], multicast=False)
        if row["N"] < 4096:
            assert round(t / 1e6, 2) == row["traffic_mb"]
        else:
            assert round(t / 1e9, 2) == 1.64
        # printed amplification = decimal MB over the "98 MB" label
        assert round(t / 1e6 / 98, 2) == pytest.approx(row["printed_amplification"], abs=0.011)
        if prev is not None:
            assert t == 2 * prev
        prev = t
        # multicast with cluster >= ceil(N/tile_n) restores 1x
        need = Pt.consumers_per_host_row(row["N"], g["tile_n"])
        assert Pt.host_traffic(host_bytes, row["N"], g["tile_n"], multicast=True, cluster_max=need) == host_bytes
        assert Pt.host_traffic(host_bytes, row["N"], g["tile_n"], multicast=True, cluster_max=2) <= t


def test_balanced_ranges():
    for R in range(0, 300, 7):
        for n in range(1, 40):
            rs = Pt.balanced_ranges(R, n)
            sizes = [b - a for a, b in rs]
            assert sum(sizes) == R and max(sizes) - min(sizes) <= 1
            assert all(rs[i][1] == rs[i + 1][0] for i in range(n - 1))
    rr = Pt.linear_row_ranges(4096, 32, 2, 146)
    assert rr[0] == ("host", 0, 16) and rr[1] == ("host", 16, 32) and rr[2][1] == 32 and rr[-1][2] == 4096


def test_attention_page_placement():
    assert Pt.host_pages_prefix(2048, 0.5, 16) == 1024
    assert Pt.host_pages_prefix(10, 0.0, 4) == 0
    assert Pt.host_pages_prefix(10, 1.0, 4) == 10
    assert Pt.batch_split_host_requests(8, 0.25) == 2


def test_kv_place_chunk_major_pins():
    """oracle.partition.kv_place_chunk_major (reading R15) against the per-request reading it
    refines and invariants it must keep: when every request has the same chunk count and the host
    units are a multiple of B, each request's host pages equal host_pages_prefix(ratio = units per
    request / chunks); host pages always form a per-request prefix, at most one chunk apart between
    requests (chunk-major = oldest first across requests), pool indices are a permutation, and
    host_tokens counts exactly the cached tokens on host pages."""
    import numpy as np
    from fractions import Fraction
    g = np.random.default_rng(77)
    for _ in range(300):
        B = int(g.integers(1, 7))
        page = int(g.choice([16, 64]))
        cp = int(g.integers(1, 4))
        L = int(g.integers(1, 900))
        pages = -(-L // page)
        chunks = -(-pages // cp)
        k = int(g.integers(0, chunks + 1))
        table, nh, ng, ht = Pt.kv_place_chunk_major([L] * B, page, pages + 1, cp, k * B)
        for b in range(B):
            host = [(e & 0x80000000) != 0 for e in table[b]]
            assert sum(host) == Pt.host_pages_prefix(pages, Fraction(k, chunks) if chunks else 0, cp)
    for _ in range(300):
        B = int(g.integers(1, 7))
        page, cp = 16, int(g.integers(1, 4))
        Ls = [int(g.integers(0, 300)) for _ in range(B)]
        max_pages = max(1, max(-(-L // page) for L in Ls))
        n_chunks = [-(-(-(-L // page)) // cp) for L in Ls]
        hu = int(g.integers(0, sum(n_chunks) + 1))
        table, nh, ng, ht = Pt.kv_place_chunk_major(Ls, page, max_pages, cp, hu)
        hc = []
        tok = 0
        for b in range(B):
            host = [(e & 0x80000000) != 0 for e in table[b]]
            hp = sum(host)
            assert host == [True] * hp + [False] * (max_pages - hp)  # prefix
            hc.append(-(-hp // cp))
            tok += min(hp * page, Ls[b])
        assert sum(hc) == hu and ht == tok
        full = [c for c, n in zip(hc, n_chunks) if c < n]  # requests not entirely on the host
        if full:
            assert max(full) - min(full) <= 1
        idx_h = sorted(e & 0x7FFFFFFF for row in table for e in row if e & 0x80000000)
        idx_g = sorted(e for row in table for e in row if not e & 0x80000000)
        assert idx_h == list(range(nh)) and idx_g == list(range(ng))


def _random_replace_case(g):
    """A decode-step re-placement: B requests grow from Ls0 to Ls1 tokens, host units old -> new."""
    B = int(g.integers(1, 6))
    page = int(g.choice([16, 64]))
    cp = int(g.integers(1, 4))
    Ls0 = [int(g.integers(1, 400)) for _ in range(B)]
    Ls1 = [L + int(g.integers(0, 200)) for L in Ls0]
    max_pages = max(-(-L // page) for L in Ls1) + int(g.integers(0, 2))
    ch0 = sum(-(-(-(-L // page)) // cp) for L in Ls0)
    ch1 = sum(-(-(-(-L // page)) // cp) for L in Ls1)
    hu0 = int(g.integers(0, ch0 + 1))
    hu1 = int(g.integers(0, ch1 + 1))
    return B, page, cp, Ls0, Ls1, max_pages, hu0, hu1


def test_kv_replace_pins():
    """oracle.partition.kv_replace (reading R23: KV placement across decode steps) against what it
    must keep: (1) every entry's tier is the fresh chunk-major placement's for the new lengths and
    host units; (2) an entry whose tier is unchanged keeps its slot, and the moves are exactly the
    tier changes; (3) no two entries share a slot of a pool, and every move writes a slot the OLD
    table did not use (copies never overwrite live data); (4) replaying the moves on simulated pools
    leaves every cached page's content readable through the new table; (5) unchanged lengths and
    units give no moves. Plus a worked example by hand."""
    import numpy as np
    HOST = 0x80000000
    # worked example: 2 requests of 128 / 200 tokens, page 64, 1-page chunks, 1 host unit (request
    # 0's page 0); they grow to 192 / 256 tokens and get 4 host units = chunks 0 and 1 of both
    # requests. Old HBM slots: request 0 pages 1-4 -> 0-3, request 1 pages 0-4 -> 4-8. Free host
    # slots 1, 2, 3, ... go to (0, 1), (1, 0), (1, 1) in (request, page) order.
    t0, _, _, _ = Pt.kv_place_chunk_major([128, 200], 64, 5, 1, 1)
    new, moves = Pt.kv_replace(t0, [192, 256], 64, 5, 1, 4, 10, 10)
    assert new == [[HOST | 0, HOST | 1, 1, 2, 3], [HOST | 2, HOST | 3, 6, 7, 8]]
    assert moves == [(0, 1, 0, HOST | 1), (1, 0, 4, HOST | 2), (1, 1, 5, HOST | 3)]
    g = np.random.default_rng(91)
    for _ in range(300):
        B, page, cp, Ls0, Ls1, max_pages, hu0, hu1 = _random_replace_case(g)
        old, nh0, ng0, _ = Pt.kv_place_chunk_major(Ls0, page, max_pages, cp, hu0)
        cap_h, cap_g = B * max_pages, B * max_pages
        new, moves = Pt.kv_replace(old, Ls1, page, max_pages, cp, hu1, cap_h, cap_g)
        fresh, _, _, _ = Pt.kv_place_chunk_major(Ls1, page, max_pages, cp, hu1)
        changed = []
        for b in range(B):
            for p in range(max_pages):
                assert bool(new[b][p] & HOST) == bool(fresh[b][p] & HOST)          # (1)
                if bool(old[b][p] & HOST) == bool(new[b][p] & HOST):
                    assert new[b][p] == old[b][p]                                  # (2)
                else:
                    changed.append((b, p, old[b][p], new[b][p]))
        assert changed == moves                                                    # (2)
        flat = [e for row in new for e in row]
        assert len(set(flat)) == len(flat)                                         # (3)
        old_used = {e for row in old for e in row}
        assert all(dst not in old_used for _, _, _, dst in moves)                  # (3)
        pools = {}                                                                 # (4)
        for b in range(B):
            for p in range(max_pages):
                pools[old[b][p]] = (b, p)
        for _, _, src, dst in moves:
            pools[dst] = pools[src]
        for b in range(B):
            for p in range(-(-Ls0[b] // page)):
                assert pools[new[b][p]] == (b, p)
        same, moves2 = Pt.kv_replace(old, Ls0, page, max_pages, cp, hu0, cap_h, cap_g)
        assert same == old and moves2 == []                                        # (5)
    with pytest.raises(ValueError):  # the host pool is full
        Pt.kv_replace(t0, [192, 256], 64, 5, 1, 4, 2, 10)


def test_kv_host_units_keep_ratio_pins():
    """round-half-up of x * n in exact rationals (reading R23 with R6's rounding): exact halves go up,
    the ratio is kept exactly when n scales by an integer, never more than n units, 0 of 0."""
    assert Pt.kv_host_units_keep_ratio(1, 4, 6) == 2        # 1.5 -> 2
    assert Pt.kv_host_units_keep_ratio(1, 4, 5) == 1        # 1.25 -> 1
    assert Pt.kv_host_units_keep_ratio(3, 8, 12) == 5       # 4.5 -> 5
    assert Pt.kv_host_units_keep_ratio(0, 7, 100) == 0
    assert Pt.kv_host_units_keep_ratio(7, 7, 9) == 9
    assert Pt.kv_host_units_keep_ratio(0, 0, 5) == 0
    for h0 in range(0, 9):
        for k in range(1, 5):
            assert Pt.kv_host_units_keep_ratio(h0, 8, 8 * k) == h0 * k


def test_calib_choice_pins():
    """oracle.partition.calib_choice (reading R24) on an end-to-end sweep shaped like the paper's
    Fig. 6: a balanced split op of C bytes at r* = B_h / (B_g + B_h) takes
    max(HBM part / B_g(n, w), host part / B_h(n, w)); B_h rises with host SMs x window until the link
    saturates, B_g degrades past 8 requests in flight (the GH200 congestion). The choice is the
    cheapest point within the tolerance of the fastest; exact ties go to the first index."""
    n_host, window = [1, 2, 4, 8, 16], [1, 2, 4, 8]
    Bg, Bh = 6500.0, 50.0
    r = Bh / (Bg + Bh)
    bh = lambda n, w: min(Bh, 7.0 * n * w)
    bg = lambda n, w: Bg - (0.0 if n * w <= 8 else 30.0 * (n * w - 8))
    t = lambda n, w: max((1 - r) / bg(n, w), r / bh(n, w))  # per byte of the op
    tab = [[((1 - r) / t(n, w), r / t(n, w)) for w in window] for n in n_host]
    i, j = Pt.calib_choice(tab, n_host, window, 0.0)
    assert (n_host[i], window[j]) == (1, 8)     # 8 in flight saturate the link, no congestion
    i, j = Pt.calib_choice(tab, n_host, window, 0.2)
    assert (n_host[i], window[j]) == (1, 8)     # everything below 8 in flight loses > 20%
    i, j = Pt.calib_choice(tab, n_host, window, 0.5)
    assert (n_host[i], window[j]) == (1, 4)     # 28 of 50 GB/s: the op at 3668 of 6550 is within 50%
    tab2 = [[(100.0, 0.0), (100.0, 0.0)], [(100.0, 0.0), (100.0, 0.0)]]
    assert Pt.calib_choice(tab2, [2, 2], [3, 3], 0.0) == (0, 0)    # ties: first index
    assert Pt.calib_choice([[(1.0, 1.0), (2.0, 0.0)]], [4], [8, 2], 0.0) == (0, 1)  # smaller window value


def test_linear_splitk_items_cover_rows():
    """oracle.partition.linear_splitk_items: every row of each tier is owned by exactly `splits`
    CTAs of that tier, in blocks of `block` rows (the last short), host tier first."""
    for M, h, S in ((7168, 1024, 2), (1280, 128, 13), (1000, 0, 3), (300, 300, 4), (129, 1, 5)):
        items = Pt.linear_splitk_items(M, h, S, 128)
        cover = [0] * M
        for tier, a, b in items:
            assert (tier == "host") == (b <= h) and b - a <= 128 and a < b
            for r in range(a, b):
                cover[r] += 1
        assert cover == [S] * M
        assert [t for t, _, _ in items] == sorted([t for t, _, _ in items], key=lambda t: t != "host")
