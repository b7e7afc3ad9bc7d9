"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel and per grid size."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, gi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = collections.defaultdict(float)
cnt = collections.Counter()
by_grid = collections.defaultdict(float)
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    tot[name] += us
    cnt[name] += 1
    by_grid[(name, r[gi])] += us
T = sum(tot.values())
print(f"{'kernel':55s} {'n':>5s} {'total us':>10s} {'share':>6s} {'avg us':>9s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:55]:55s} {cnt[k]:5d} {v:10.1f} {v / T * 100:5.1f}% {v / cnt[k]:9.2f}")
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
if "-g" in sys.argv:
    for (k, gsz), v in sorted(by_grid.items(), key=lambda x: -x[1])[:25]:
        print(f"  {k[:45]:45s} grid {gsz:>16s} {v:9.1f} us")
