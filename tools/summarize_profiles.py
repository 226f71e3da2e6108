"""Turn a round's raw ncu outputs (gpurun_out/, scratch) into the committed summaries under
profiles/<round>/: the per-kernel-family launch table of one timed decode step (duration share
and DRAM bytes per launch) and linear_traffic.json, which bench.py reads for roofline.traffic
(DRAM read+write bytes per dak_linear launch, averaged over the step's linear launches)."""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_table(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            h, body = r, rows[i + 1:]
            break
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
    per = collections.OrderedDict()
    for r in body:
        if len(r) > vi:
            per.setdefault((r[0], r[ki]), {})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    return per


def family(name):
    return re.sub(r"\(.*", "", name).replace("void ", "").split("::")[-1]


def main(rnd="r02", csv_name="launches_opt.csv", workload="opt-30b-decode-b8-ctx64", out_rnd=None):
    out_dir = os.path.join(ROOT, "profiles", out_rnd or rnd)
    os.makedirs(out_dir, exist_ok=True)
    src = os.path.join(ROOT, "gpurun_out", rnd, csv_name)
    per = launch_table(src)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    lin_n, lin_bytes = 0, 0.0
    for (_, name), m in per.items():
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[family(name)]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += b
        if re.search(r"split_linear|umma_linear|umma_swap", name):
            lin_n += 1
            lin_bytes += b
    tot = sum(a[1] for a in agg.values())
    lines = [f"# one timed {workload} decode step ({len(per)} launches), ncu --metrics gpu__time_duration.sum,"
             "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (serialised, cold L2:",
             "shares are meaningful, absolute times are not the graph's); tools/profile_round.sh",
             f"{'launches':>8} {'total_us':>10} {'share':>6} {'mean_us':>8} {'dram_MB/launch':>15}  kernel"]
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{c:8d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {t / c / 1e3:8.2f} {b / c / 1e6:15.2f}  {k}")
    lines.append(f"total {tot / 1e3:.1f} us")
    open(os.path.join(out_dir, f"step_launches_{workload}.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(dict(source=f"gpurun_out/{rnd}/{csv_name} (ncu, one timed step of {workload})", linear_launches=lin_n,
                   dram_bytes_per_launch=round(lin_bytes / max(lin_n, 1))),
              open(os.path.join(out_dir, f"linear_traffic_{workload}.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
