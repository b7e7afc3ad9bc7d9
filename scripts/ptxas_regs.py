"""Parse `nvcc -Xptxas -v` output (stdin): demangled entry, registers, spill bytes."""
import re, subprocess, sys
cur = None
rows = []
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur:
        sp = (int(m.group(1)), int(m.group(2)))
        rows.append([cur, None, sp])
    m = re.search(r"Used (\d+) registers", ln)
    if m and rows and rows[-1][1] is None:
        rows[-1][1] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for (mang, regs, sp), nm in zip(rows, names):
    if pat in nm:
        nm = re.sub(r"mgb::\(anonymous namespace\)::", "", nm).replace("(mgb::StreamArgs)", "")
        print(f"{regs:4d} regs  spill {sp[0]:5d}/{sp[1]:5d}  {nm}")
