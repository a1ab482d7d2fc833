"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel: launches, total ms,
share of the summed kernel time.  usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
    name = r[ki].split("(")[0][:60]
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"launches {sum(cnt.values())} total kernel ms {all_ms:.1f}")
for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{ms:10.2f} ms {100 * ms / all_ms:6.1f}% {cnt[name]:6d}  {name}")
