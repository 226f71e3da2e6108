"""Join tools/link_counters.py's cases with the ncu CSV of the same run (one captured launch per
case, same order) and print measured link / DRAM bytes against the algorithmic ones.

  python tools/summarize_link.py gpurun_out/link_cases.jsonl gpurun_out/link_ncu.csv > profiles/r02/link_counters.txt
"""
from __future__ import annotations

import csv
import json
import sys


def load_ncu(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        val = d["Metric Value"].replace(",", "")
        unit = d.get("Metric Unit", "")
        try:
            v = float(val)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20, "GB": 1 << 30,
                 "ns": 1e-9, "us": 1e-6, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "sector": 1}.get(unit, 1)
        e = out.setdefault(key, dict(kernel=d["Kernel Name"]))
        e[d["Metric Name"]] = v * scale
    return [out[k] for k in sorted(out)]


def main():
    cases = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
    launches = load_ncu(sys.argv[2])
    print(f"# {len(cases)} cases, {len(launches)} captured launches (one per case, in order)")
    print("case | kernel | host B (alg) | pcie read B | sysmem sectors x32 B | link/host | DRAM read B | HBM alg B | us")
    for c, m in zip(cases, launches):
        pr = m.get("pcie__read_bytes.sum", float("nan"))
        ss = m.get("syslts__t_sectors_aperture_sysmem.sum", float("nan")) * 32
        dr = m.get("dram__bytes_read.sum", float("nan"))
        t = m.get("gpu__time_duration.sum", float("nan")) * 1e6
        hb = c["host_bytes"]
        print(f"{c['case']} | {m['kernel'][:40]} | {hb:.0f} | {pr:.0f} | {ss:.0f} | "
              f"{(pr / hb if hb else float('nan')):.3f} / {(ss / hb if hb else float('nan')):.3f} | {dr:.0f} | "
              f"{c['hbm_bytes']:.0f} | {t:.1f}")


if __name__ == "__main__":
    main()
