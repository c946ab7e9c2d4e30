"""Summarise an ncu launch list (gpu__time_duration.sum, --csv) by kernel.

    python tools/summarize_launches.py gpurun_out/r1_launches.csv > profiles/r1_launches_summary.txt
"""
import collections
import csv
import re
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h, data = rows[0], rows[1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in data:
        name = re.sub(r"^void ", "", r[ik])
        cut = name.rfind(">(")
        name = name[: cut + 1] if cut > 0 else re.sub(r"\(.*", "", name)
        name = name.replace("(int)", "")
        us = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
        tot += us
    print(f"# {path}: {len(data)} launches, {tot / 1e3:.2f} ms of kernel time "
          f"(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)")
    print(f"{'kernel':72s} {'launches':>8s} {'total us':>12s} {'share':>7s} {'avg us':>10s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:72]:72s} {n:8d} {t:12.1f} {100 * t / tot:6.2f}% {t / n:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
