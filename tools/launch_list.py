"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by
kernel (tools only). usage: python tools/launch_list.py launches.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
unit = rows[1][h.index("Metric Unit")] if "Metric Unit" in h else ""
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"^.*::", "", name) if "<" not in name else name.split("::")[-1]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if unit == "nsecond" or unit == "ns" else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
n = sum(v[0] for v in agg.values())
print(f"# {n} launches, {tot:.1f} us total")
print(f"{'kernel':50s} {'launches':>8s} {'sum_us':>12s} {'share':>7s} {'avg_us':>9s}")
for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:50]:50s} {c:8d} {s:12.1f} {s / tot:7.3f} {s / c:9.2f}")
