"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel count / total / mean device time, optionally only the last N sweeps'
launches (skip setup)."""
import csv
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lines = [l for l in open(path) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
rows = rows[skip:]
agg = OrderedDict()
total = 0.0
for r in rows:
    name = r["Kernel Name"]
    name = re.sub(r"\(.*", "", name).replace("cpdb::", "").replace("<unnamed>::", "")
    name = re.sub(r"^.*::", "", name) if "::" in name else name
    t = float(r["Metric Value"]) / 1e3
    a = agg.setdefault(name + " " + r["Grid Size"], [0, 0.0])
    a[0] += 1
    a[1] += t
    total += t
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:10.1f} us {100 * t / total:5.1f}%  n={n:4d}  mean={t / n:8.1f} us  {k}")
print(f"total {total:.1f} us over {len(rows)} launches")
