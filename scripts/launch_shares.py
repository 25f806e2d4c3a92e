"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel.

    python scripts/launch_shares.py launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i + 1
        break
ki, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= mv:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':<55} {'launches':>8} {'total_ms':>9} {'share':>6} {'avg_us':>8}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:55]:<55} {c:8d} {t / 1e3:9.2f} {100 * t / tot:5.1f}% {t / c:8.1f}")
print(f"{'total':<55} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:9.2f}")
