"""A/B of the streaming kernels on a bench config: per-level PRE / POST pass times
(mgb_time_pass, CUDA events) and the whole 10-cycle solve, per kernel kind."""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2102_12071_b200 import _lib, device as dv
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
kinds = [int(k) for k in (sys.argv[2] if len(sys.argv) > 2 else "2,3").split(",")]
h, f_host, info = bench.build_problem(cfg, 0)
nu, cycles = info["nu"], info["cycles"]
f = torch.from_numpy(np.ascontiguousarray(f_host[0])).cuda()
n = f.shape[0]
res = {}
us = {}
for kind in kinds:
    h.set_stream_kernel(kind)
    w = h.acquire_work()
    row = {}
    for l in range(min(4, h.depth - 1)):
        rows, cols = h.level_info(l)[:2]
        fl = f if l == 0 else torch.randn(rows, cols, dtype=torch.float64, device="cuda")
        ut = torch.zeros_like(fl)
        for p in (0, 1):
            ms = C.c_double()
            _lib.call("mgb_time_pass", h.handle, w, l, p, nu, dv.ptr(fl), dv.ptr(ut), 20, C.byref(ms), dv.stream(fl))
            row[f"L{l}{'PRE' if p == 0 else 'POST'}_us"] = round(ms.value * 1e3, 1)
    h.release_work(w)
    u = torch.zeros_like(f)
    hist = torch.empty(1, cycles + 1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        h.run_cycles(f, u, cycles, nu, nu, history=hist, u_zero=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        h.run_cycles(f, u, cycles, nu, nu, history=hist, u_zero=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    row["solve_ms"] = round(ms, 4)
    row["unknowns_per_s"] = n * n * cycles / (ms * 1e-3)
    row["hist_last"] = float(hist[0, -1])
    us[kind] = u.clone()
    res[kind] = row
    print(kind, json.dumps(row), flush=True)
if len(kinds) > 1:
    a, b = us[kinds[0]], us[kinds[1]]
    print("u bitwise equal:", bool(torch.equal(a, b)), "max diff", float((a - b).abs().max()))
