"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel family.

usage: python tools/summarize_launches.py gpurun_out/launches.csv > profiles/rNN/launch_summary.txt
Per-launch ncu times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import collections
import csv
import re
import sys


def short(name):
    name = name.replace("<unnamed>::", "")
    name = re.sub(r"^void\s+", "", name)
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = name.replace("sc::", "")
    m = re.match(r"([A-Za-z_0-9:]+)(<[^()]*>)?", name)
    base = m.group(1) if m else name
    tmpl = m.group(2) or "" if m else ""
    return base + tmpl


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot/1e3:.1f} ms total (cold-cache, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>14s} {'avg_us':>12s} {'share':>8s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:60s} {c:8d} {t:14.1f} {t/c:12.2f} {100*t/tot:7.3f}%")


if __name__ == "__main__":
    main(sys.argv[1])
