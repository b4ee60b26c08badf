"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    n = r[ki].split("(")[0]
    n = n.replace("void ", "").split("<")[0]
    if "k_init_tables" in n:
        continue
    agg[n][0] += 1
    agg[n][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'us/launch':>10s} {'share':>6s}")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:40s} {c:8d} {t / 1e3:10.1f} {t / c / 1e3:10.1f} {100 * t / tot:5.1f}%")
print(f"total {tot / 1e3:.1f} us")
