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
