"""Top stalled SASS instructions of one kernel launch with their stall reasons.
    python scripts/ncu_stalls.py REPORT LAUNCH_INDEX [top]"""
import csv, subprocess, sys
rep, idx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1][:120])
hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ia = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda v: int(v) if v.isdigit() else 0  # noqa: E731
tot = sum(num(r[ia]) for r in data)
agg = {h: sum(num(r[hdr.index(h)]) for r in data) for h in reasons}
print("total samples", tot, " ", ", ".join(f"{h[6:]} {v * 100 // max(tot, 1)}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
addr = [r[0] for r in data]
for r in sorted(data, key=lambda r: -num(r[ia]))[:top]:
    i = addr.index(r[0])
    why = sorted(((num(r[hdr.index(h)]), h[6:]) for h in reasons), reverse=True)[:2]
    prev = data[i - 1][1].strip()[:40] if i else ""
    print(f"{r[0][-5:]} {num(r[ia]) * 100 / tot:5.1f}% {why}  {r[1].strip()[:60]:60s} | prev: {prev}")
