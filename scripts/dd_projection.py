"""Projection (NOT a measurement) of the decomposed solve's per-rank time on N GPUs from
single-GPU timings: all N parts run one after another on this GPU (virtual backend: halos by
device copies), the replicated coarse cycle once.

    T_virtual(N) = sum over parts of their fine-level passes + T_coarse + copies
    T_rank(N)   ~= (T_virtual(N) - T_coarse) / N + T_coarse          (+ exposed exchange time)
    E(N)         = T_single / (N * T_rank(N))

T_coarse: the agglomerated levels' cycle (level La downwards), timed with mgb_vcycle.  The
exchange term is reported separately as latency-bound and bandwidth-bound estimates: the
schedule overlaps the exchanges with the interior launches, so the exposed part lies between
zero and that figure.  Usage: python scripts/dd_projection.py c5 2,4,8"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2102_12071_b200 import _lib, dd, device as dv

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5"
parts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
cfg = bench.CONFIGS[cfg_name]
h, f_host, info = bench.build_problem(cfg_name, 0)
n, nu, cycles = cfg["n"], cfg["nu"], cfg["cycles"]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


f = torch.from_numpy(np.ascontiguousarray(f_host[0])).cuda()
u = torch.zeros_like(f)
hist = torch.empty((1, cycles + 1), dtype=torch.float64, device="cuda")
t_single = timed(lambda: h.run_cycles(f, u, cycles, nu, nu, history=hist, u_zero=True))
del u
out = {"config": cfg_name, "ms_per_step_single": t_single, "rows": []}
for N in parts:
    s = dd.DecomposedSolver(h, N, local=True, agglomerate_rows=1023)
    for p in range(N):
        r0, r1 = s.rows(p)
        s.set_rhs(p, f[r0:r1].contiguous())
    hd = torch.empty(cycles + 1, dtype=torch.float64, device="cuda")
    t_virtual = timed(lambda: s.run_cycles(cycles, nu, nu, True, hd))
    sent, steps = s.stats()
    La = s.distributed_levels
    # the agglomerated coarse cycle alone
    w = h.acquire_work()
    rows, cols = h.level_info(La)[:2]
    fc = torch.randn(rows, cols, dtype=torch.float64, device="cuda")
    uc = torch.zeros_like(fc)
    t_coarse = cycles * timed(lambda: _lib.call("mgb_vcycle", h.handle, w, La, dv.ptr(fc), dv.ptr(uc), nu, nu, dv.stream(fc)), reps=20)
    h.release_work(w)
    t_rank = (t_virtual - t_coarse) / N + t_coarse
    # exchange estimates per step for one interior rank: latency 20 us per exchange step,
    # bandwidth: its share of the bytes at 400 GB/s effective NVLink per direction
    t_lat = steps * 20e-3
    t_bw = (sent / N) / 400e9 * 1e3
    out["rows"].append({"n_gpus": N, "ms_virtual_all_parts": t_virtual, "ms_coarse_replicated": t_coarse,
                        "ms_rank_projected": t_rank, "efficiency_projected_no_exchange": t_single / (N * t_rank),
                        "exchange_steps_per_step": steps, "exchange_ms_if_fully_exposed": t_lat + t_bw,
                        "efficiency_projected_exchange_exposed": t_single / (N * (t_rank + t_lat + t_bw)),
                        "history_last": float(hd[-1])})
    print(json.dumps(out["rows"][-1]), flush=True)
    del s
    torch.cuda.empty_cache()
out["history_last_single"] = float(hist[0, -1])
print(json.dumps(out))
