"""Per-source-line instruction counts / stall samples of one kernel in an ncu report:
    python scripts/ncu_lines.py REPORT LAUNCH_INDEX [top]"""
import collections, csv, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr = None, None
per_line = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
cur_file = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    v = r[hdr.index("Instructions Executed")]
    ie = int(v) if v.isdigit() else 0
    v = r[hdr.index("Warp Stall Sampling (All Samples)")]
    st = int(v) if v.isdigit() else 0
    sass = r[3].strip()
    key = (cur_file, ln)
    e = per_line[key]
    e[0] += ie
    e[1] += st
    if sass:
        op = sass.split()
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        e[2][o.split(".")[0]] += ie
    if not e[3]:
        e[3] = r[1].strip()[:70]
print(fname)
tot = sum(v[0] for v in per_line.values())
tst = sum(v[1] for v in per_line.values())
print("total warp instructions", tot, "stall samples", tst)
for (f, ln), (ie, st, ops, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:4d} {ie / tot * 100:5.1f}% inst {st / max(tst,1) * 100:5.1f}% stall  {src:70s} "
          + ",".join(f"{o}:{n * 100 // max(ie, 1)}" for o, n in ops.most_common(4)))
