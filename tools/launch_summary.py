"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
launches, average us and share per kernel.  usage: launch_summary.py FILE.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= vi or not r[vi].replace(".", "").replace(",", "").isdigit():
        continue
    name = r[ki].split("(")[0]
    if name.startswith("void "):
        name = name[5:]
    v = float(r[vi].replace(",", "")) * (1e-3 if r[ui] in ("ns", "nsecond") else 1e3 if r[ui] in ("ms", "msecond") else 1.0)
    tot[name] += v
    cnt[name] += 1
scale = 1.0  # microseconds
all_ = sum(tot.values())
print(f"{'kernel':60s} {'n':>4s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:4d} {tot[k] / cnt[k] * scale:9.1f} {100 * tot[k] / all_:5.1f}%")
