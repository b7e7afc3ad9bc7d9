"""Print key metrics, stall reasons and the instruction mix of an ncu report."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "local_load", "smsp__sass_inst_executed_op_local_ld.sum"]
for r in rows[2:]:
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:72s} {r[i][:70]:>24s} {units[i]}")
    st = [(float(r[i].replace(",", "") or 0), h) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in h and r[i]]
    for v, h in sorted(st, reverse=True)[:7]:
        print(f"    {h[33:]:60s} {v:.0f}")
    print()
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
blocks, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        blocks.append(cur)
    elif r and r[0] == "Address":
        hdr = r
    elif r and cur is not None and hdr:
        cur[1].append(r)
for name, data in blocks:
    si, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    for r in data:
        op = r[si].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(r[ie] or 0)
    tot = sum(c.values())
    print(name[:100], "instructions", tot)
    print("   ", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in c.most_common(16)))
