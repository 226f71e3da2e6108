"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel-family count,
total and mean duration over the LAST `--tail` launches (one decode step)."""
import argparse
import collections
import csv
import re


def load(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, body = r, rows[i + 1:]
            break
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    out = []
    for r in body:
        if len(r) > vi and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            out.append((r[ki], r[gi], float(r[vi].replace(",", ""))))
    return out


def family(name):
    m = re.match(r"(?:void )?(?:dak::)?(?:\w+::)?(\w+)(?:<([^>]*)>)?", name)
    return (m.group(1) + (f"<{m.group(2)}>" if m.group(2) else "")) if m else name[:50]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tail", type=int, default=0)
    a = ap.parse_args()
    L = load(a.csv)
    if a.tail:
        L = L[-a.tail:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, g, t in L:
        k = family(n)
        agg[k][0] += 1
        agg[k][1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(L)}  total {tot / 1e3:.1f} us (ncu: serialised, cold-cache)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:5d}  {t / 1e3:10.1f} us  {100 * t / tot:5.1f}%  mean {t / c / 1e3:8.2f} us  {k}")
