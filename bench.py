"""Benchmark: unknowns/s per V-cycle (fp64) of the learned-smoother multigrid solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Workload (N = 1): BASELINE.json config 2 — rotated anisotropic Laplacian
(reference FD stencil, eps = 1e-3, theta = pi/4) on a 4095^2 interior grid,
11 levels, Galerkin coarse operators, per-point smoother kernels from the
seeded conv inference net (tests/golden/net_conv_c2.json: the reference's own
SURVEY-G4 training recipe run at the config's theta/eps),
b ~ U[-1, 1] (seed 1), u0 = 0.  One step = one 10-cycle V(2,2) solve including
the per-cycle residual history (as hierarchy.solve times it).  Multi-GPU (torchrun):
every rank solves its own copy of the problem (weak scaling, no data-path
collective); the job value is the sum over ranks of unknowns / max-over-ranks time.

`--impl reference` times the CPU oracle port of the reference algorithm (NumPy,
oracle/mg_oracle.py) on a bounded sample of the same workload (see cpu_sample()).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, theta, eps, levels, nu, cycles, rhs seed)
    "c2": (4095, math.pi / 4, 1e-3, 11, 2, 10, 1),
    "c1": (255, math.pi / 6, 0.01, 7, 2, 20, 0),
}
# inference net per config: the SURVEY G4 training recipe run by the reference at the
# config's own (theta, eps) (tests/golden/make_golden.py)
NETS = {"c2": "net_conv_c2.json", "c1": "net_conv.json"}
# algorithmic bytes of one pass, per-point fp64 model
SWEEP_BYTES_PER_POINT = 168          # read u, f, A(9), M(9); write u
CPU_SAMPLE_N = 1023                  # bounded CPU sample: same operator family at 1023^2


def cycle_bytes_per_fine_unknown(n, levels, nu1, nu2):
    """sum_l N_l (168 (nu1+nu2) - 80 [l>=1] + 104) + 16 N_{l+1}, + 16 N_L."""
    sizes = []
    m = n
    for _ in range(levels):
        sizes.append(m * m)
        m //= 2
    tot = 0.0
    for l in range(levels - 1):
        tot += sizes[l] * (168 * (nu1 + nu2) - 80 * (l >= 1) + 104) + 16 * sizes[l + 1]
    tot += 16 * sizes[-1]
    return tot / sizes[0]


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def ncu_traffic():
    """DRAM bytes per launch of the level-0 PRE pass from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get("pre_dram_bytes_per_launch"), d
        except Exception:
            pass
    return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def build_problem(cfg_name, device):
    import paper_2102_12071_b200 as mg
    from paper_2102_12071_b200 import problems as gen
    n, theta, eps, levels, nu, cycles, seed = CONFIGS[cfg_name]
    A = gen.rotated_fd(n, theta, eps)
    f = gen.uniform_rhs(n, seed)
    net = mg.load_model(os.path.join(ROOT, "paper_2102_12071_b200", "data", NETS[cfg_name]))
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), levels, device=device)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    mg.equip_inferred(h, net)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del A
    return h, f, dict(n=n, theta=theta, eps=eps, levels=levels, nu=nu, cycles=cycles, seed=seed,
                      setup_rap_lu_s=t1 - t0, setup_infer_s=t2 - t1)


def cpu_sample(cfg_name, steps=1, warmup=0):
    """Oracle port (NumPy, single thread) on a bounded sample: the config's operator
    family at CPU_SAMPLE_N^2 (levels scaled to reach 3x3), V(nu, nu) cycles with
    the history residual, timed like hierarchy.solve (setup excluded)."""
    from oracle import mg_oracle as mo
    from paper_2102_12071_b200 import problems as gen
    n0, theta, eps, levels0, nu, cycles, seed = CONFIGS[cfg_name]
    n = min(n0, CPU_SAMPLE_N)
    levels = gen.levels_for(n)
    A = gen.rotated_fd(n, theta, eps)
    f = gen.uniform_rhs(n, seed)
    t0 = time.perf_counter()
    h = mo.build_hierarchy(A, levels)
    mo.equip_inferred(h, mo.load_net_json(os.path.join(ROOT, "paper_2102_12071_b200", "data", NETS[cfg_name])))
    setup = time.perf_counter() - t0
    u = np.zeros((n, n))
    fn = float(np.linalg.norm(f))
    times = []
    for s in range(warmup + steps):
        t = time.perf_counter()
        u = mo.v_cycle(h, 0, f, u, nu, nu)
        _ = float(np.linalg.norm(f - mo.apply_stencil(A, u))) / fn
        dt = time.perf_counter() - t
        if s >= warmup:
            times.append(dt)
    per_cycle = float(np.mean(times))
    return {"value": n * n / per_cycle, "unit": "unknowns/s", "cores": 1, "kind": "port",
            "sample": f"oracle/mg_oracle.py (NumPy, 1 thread) V({nu},{nu}) cycle + history residual on the "
                      f"config's operator at {n}^2 ({levels} levels), {len(times)} cycle(s) timed, "
                      f"setup {setup:.1f}s excluded; cpu {cpu_model()}",
            "per_cycle_s": per_cycle}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except Exception:
        pass
    return f"{os.cpu_count()} cpus"


def run_reference(args):
    world, rank, local = dist_init()
    if rank != 0:
        return 0
    n, theta, eps, levels, nu, cycles, seed = CONFIGS[args.config]
    s = cpu_sample(args.config, steps=max(1, args.steps), warmup=min(args.warmup, 1))
    line = {"metric": "unknowns/sec per V-cycle (fp64)", "value": s["value"], "unit": "unknowns/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s["per_cycle_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators)", "impl": "reference",
            "config": {"workload": f"{args.config}: rotated FD eps={eps} theta={theta:.4f} {n}^2 V({nu},{nu}) "
                                   f"learned conv smoother", "sample_n": min(n, CPU_SAMPLE_N)},
            "cpu_baseline": {k: s[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": s["value"], "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2102_12071_b200 as mg
    from paper_2102_12071_b200 import _lib
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    h, f_host, info = build_problem(args.config, local)
    n, levels, nu, cycles = info["n"], info["levels"], info["nu"], info["cycles"]
    f = torch.from_numpy(f_host).to(dev)
    u = torch.zeros_like(f)
    hist = torch.empty((1, cycles + 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        h.run_cycles(f, u, cycles, nu, nu, history=hist, u_zero=True)
    launches_per_step = h.last_launches
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            h.run_cycles(f, u, cycles, nu, nu, history=hist, u_zero=True)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    final_hist = hist.cpu().numpy()[0]
    value = world * n * n * cycles / (ms_max * 1e-3)

    # dominant kernels: the level-0 PRE / POST phases (row-streaming passes), timed
    # live with CUDA events on the launching stream through mgb_time_pass
    import ctypes as C
    from paper_2102_12071_b200 import device as dv
    compact = all(h.storage_info(0))
    w = h.acquire_work()
    try:
        ms_pre, ms_post = C.c_double(), C.c_double()
        ut = torch.zeros_like(f)
        _lib.call("mgb_time_pass", h.handle, w, 0, 0, nu, dv.ptr(f), dv.ptr(ut), 20, C.byref(ms_pre), dv.stream(f))
        _lib.call("mgb_time_pass", h.handle, w, 0, 1, nu, dv.ptr(f), dv.ptr(ut), 20, C.byref(ms_post), dv.stream(f))
        torch.cuda.synchronize(dev)
    finally:
        h.release_work(w)
    peak, peak_kind = measured_peak()
    # algorithmic bytes per fine point: u in, f, u out (8 B each) + restricted residual
    # (PRE) or coarse correction (POST) at 8 B per coarse point; + 72 B each for A and
    # M when they are per-point planes (the reference data model)
    per_pt = 26 + (0 if compact else 144)
    pass_bytes = per_pt * n * n
    achieved = pass_bytes / (ms_pre.value * 1e-3) / 1e9
    achieved_post = pass_bytes / (ms_post.value * 1e-3) / 1e9
    traffic, _ = ncu_traffic()

    # e2e through the host-buffer C-ABI call (pinned host f in, u + history out)
    f_pin = torch.from_numpy(f_host).pin_memory()
    u_pin = torch.zeros_like(f_pin).pin_memory()
    hist_host = np.empty((1, cycles + 1))
    fh, uh = f_pin.numpy(), u_pin.numpy()
    for _ in range(2):
        h.run_cycles_host(fh, uh, cycles, nu, nu, history_host=hist_host, u_zero=True,
                          stream=dv.stream(f))
    barrier()
    e_steps = max(1, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e_steps):
        h.run_cycles_host(fh, uh, cycles, nu, nu, history_host=hist_host, u_zero=True, stream=dv.stream(f))
    e1.record(stream)
    barrier()
    e_ms = e0.elapsed_time(e1) / e_steps
    t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = world * n * n * cycles / (float(t.item()) * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(args.config, steps=1)
    if rank == 0:
        bpu = cycle_bytes_per_fine_unknown(n, levels, nu, nu)
        line = {
            "metric": "unknowns/sec per V-cycle (fp64)", "value": value, "unit": "unknowns/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators; trained seeded conv net fixture)",
            "config": {"workload": f"{args.config}: rotated FD Laplacian eps={info['eps']} theta=pi/4 "
                                   f"{n}^2, {levels} levels, V({nu},{nu}) x {cycles} cycles + history, "
                                   f"learned conv smoother (per-point fp64 A and M)",
                       "unknowns": n * n, "cycles_per_step": cycles,
                       "l2": "inputs larger than L2 (level-0 A+M = 2.4 GB)", "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm",
                         "kernel": "k_stream PRE, level 0 (2 sweeps + residual + full-weighting restriction, "
                                   "one row-streaming pass)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": pass_bytes, "launch_ms": ms_pre.value,
                         "storage": "band-class tables (A, M exact, shared memory)" if compact else "per-point planes",
                         "post": {"kernel": "k_stream POST, level 0 (prolongation + 2 sweeps)",
                                  "achieved": achieved_post, "frac": achieved_post / peak, "launch_ms": ms_post.value}},
            "cycle_model": {"survey_bytes_per_fine_unknown": bpu if not compact else 172.6,
                            "survey_model": "per-point" if not compact else "compact (SURVEY 8(d))",
                            "effective_GBps": value / world * (bpu if not compact else 172.6) / 1e9},
            "e2e": {"value": e2e_value, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * n * n,
                    "d2h_bytes_per_step": 8 * n * n + 8 * (cycles + 1)},
            "gpu_launches": int(launches_per_step * args.steps),
            "history_last": float(final_hist[-1]),
            "setup_s": {"galerkin_lu": info["setup_rap_lu_s"], "cnn_inference": info["setup_infer_s"]},
            "clocks": clk.summary(),
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
