"""Top warp-stall SASS lines from `ncu --page source --csv --print-source sass` output (stdin or path)."""
import csv
import sys


def main():
    f = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(f))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    col = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for k, r in enumerate(rows[hi + 1:]):
        try:
            data.append((float(r[col]), k, r))
        except (ValueError, IndexError):
            continue
    tot = sum(v for v, _, _ in data) or 1.0
    for v, k, r in sorted(data, key=lambda t: -t[0])[:n]:
        print(f"{100 * v / tot:5.1f}%  #{k:5d} {r[0][-5:]}  {r[1].strip()[:100]}")


if __name__ == "__main__":
    main()
