"""Benchmark: unknowns/s per V-cycle (fp64) of the learned-smoother multigrid solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Default workload (N = 1): BASELINE.json config 2 — rotated anisotropic Laplacian
(reference FD stencil, eps = 1e-3, theta = pi/4) on a 4095^2 interior grid,
11 levels, Galerkin coarse operators, per-point smoother kernels from the
seeded conv inference net (tests/golden/net_conv_c2.json: the reference's own
SURVEY-G4 training recipe run at the config's theta/eps), b ~ U[-1, 1] (seed 1),
u0 = 0.  One step = one 10-cycle V(2,2) solve including the per-cycle residual
history (as hierarchy.solve times it).

Other configs: c1 (255^2, V(2,2) x 20), c3 (8191^2 GRF 5-point variable
coefficients, per-point tables, V(2,2) x 10), c4 (256 problems at 511^2 with
random (eps, theta), V(1,1) x 10, batched hierarchy).

Multi-GPU (torchrun): the single-problem configs c2 (the default), c3 and c5 are
domain-decomposed in row blocks with NCCL halo exchange overlapped with the interior
rows and agglomerated coarse levels (strong scaling of the one problem: the N = 1
line is the same problem on one GPU); c4 splits its 256 problems across ranks (strong
scaling, no data-path collective); c1 (255^2, L2-resident) places one replica per rank.
The value is the job's unknowns / max-over-ranks device time.

`--impl reference` times the CPU oracle port of the reference algorithm (NumPy,
oracle/mg_oracle.py) on a bounded sample of the same workload on all host cores
(cpu_sample_replicas(): one single-threaded replica per core; config 4: a pool
over its independent problems).
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

# name: dict(n, levels, nu, cycles, net, batch, kind, ...)
CONFIGS = {
    "c1": dict(n=255, op="rot", theta=math.pi / 6, eps=0.01, levels=7, nu=2, cycles=20, seed=0, batch=1,
               net="net_conv.json", desc="rotated FD eps=0.01 theta=pi/6"),
    "c2": dict(n=4095, op="rot", theta=math.pi / 4, eps=1e-3, levels=11, nu=2, cycles=10, seed=1, batch=1,
               net="net_conv_c2.json", desc="rotated FD Laplacian eps=0.001 theta=pi/4"),
    "c3": dict(n=8191, op="grf", levels=12, nu=2, cycles=10, seed=2, batch=1, net="net_conv_c3.json",
               desc="-div(exp(GRF) grad u), 5-point cell-centred, corr. length 1/32, per-point tables"),
    "c4": dict(n=511, op="batch", levels=8, nu=1, cycles=10, seed=3, batch=256, net="net_conv.json",
               desc="256 rotated FD problems, log-uniform eps in [1e-3,1], theta ~ U[0,pi)"),
    "c5": dict(n=32767, op="rot_classed", theta=math.pi / 3, eps=0.01, levels=14, nu=2, cycles=10, seed=5, batch=1,
               net="net_conv_c5.json",
               desc="rotated FD eps=0.01 theta=pi/3, band-class hierarchy (no per-point tables)"),
}
# bounded CPU sample: same operator family at <= 1023^2 (MGB_CPU_SAMPLE_N: smaller, for tests)
CPU_SAMPLE_N = int(os.environ.get("MGB_CPU_SAMPLE_N", "1023"))


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


def ncu_traffic(cfg_name):
    """DRAM bytes per launch of the level-0 PRE pass from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p) and cfg_name == "c2":
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
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # wait until the sampler is producing, so the timed region is covered
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.03)  # one more sample at the end of the timed region
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


def operators(cfg, lo=0, hi=None):
    """Host inputs of a config: (A (batch, n, n, 3, 3), f (batch, n, n)) for problems [lo, hi)."""
    from paper_2102_12071_b200 import problems as gen
    n = cfg["n"]
    if cfg["op"] == "rot_classed":
        return gen.rotated_fd(1, cfg["theta"], cfg["eps"], h=1.0 / (n + 1))[0, 0], gen.uniform_rhs(n, cfg["seed"])[None]
    if cfg["op"] == "rot":
        return gen.rotated_fd(n, cfg["theta"], cfg["eps"])[None], gen.uniform_rhs(n, cfg["seed"])[None]
    if cfg["op"] == "grf":
        return gen.grf_diffusion_5pt(n, seed=cfg["seed"])[None], gen.uniform_rhs(n, cfg["seed"])[None]
    hi = cfg["batch"] if hi is None else hi
    eps, theta = gen.batch_parameters(cfg["batch"], seed=cfg["seed"])
    A = np.empty((hi - lo, n, n, 3, 3))
    f = np.empty((hi - lo, n, n))
    for k, i in enumerate(range(lo, hi)):
        A[k] = gen.rotated_fd(n, theta[i], eps[i])
        f[k] = gen.uniform_rhs(n, [4, i])
    return A, f


def build_problem(cfg_name, device, lo=0, hi=None):
    import torch
    import paper_2102_12071_b200 as mg
    cfg = CONFIGS[cfg_name]
    A, f = operators(cfg, lo, hi)
    n = cfg["n"]
    net = mg.load_model(os.path.join(ROOT, "paper_2102_12071_b200", "data", cfg["net"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cfg["op"] == "rot_classed":
        h = mg.build_hierarchy_classed(n, n, A, cfg["levels"], device=device)
    elif cfg["batch"] == 1:
        spec = mg.GridSpec(n, n, 1.0 / n if cfg["op"] == "grf" else 1.0 / (n + 1), np.ones((n, n), bool))
        h = mg.build_hierarchy(mg.StencilField(spec, A[0]), cfg["levels"], device=device)
    else:
        h = mg.build_hierarchy_batch(A, cfg["levels"], device=device)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    mg.equip_inferred(h, net)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del A
    info = dict(cfg, setup_rap_lu_s=t1 - t0, setup_infer_s=t2 - t1, local_batch=f.shape[0])
    return h, f, info


def _band(n):
    """Band index of every row / column: 0, 1 for the first two, 2 inside, 3, 4 for the last two."""
    b = np.full(n, 2)
    b[:2] = (0, 1)
    b[-2:] = (3, 4)
    return b


def oracle_hierarchy_constant(table, n, levels, net):
    """Oracle hierarchy (oracle/mg_oracle.py types) of a constant-coefficient operator
    at full size without the oracle's O(n^2 x 200 flop) setup: away from the boundary a
    constant-coefficient Galerkin chain is constant, and within two points of it it
    depends only on the band (first two rows / columns, interior, last two), so every
    level's operator is 5 x 5 class tables.  The class tables of the next level come from
    the oracle's own galerkin() on a 15 x 15 expansion (-> 7 x 7: its rows 0, 1, 3, 5, 6
    are the five bands); the conv net maps a point's own table, so the kernels are the
    net's outputs on the 25 class tables.  Levels of at most 63 points per side use the
    oracle's functions directly.  The operators equal mo.build_hierarchy's bit for bit and
    the kernels mo.equip_inferred's to one unit in the last place (BLAS blocks the net's
    last matmul differently for 25 rows; tests/test_bench_reference.py); only the timed
    cycle, which runs the oracle's v_cycle on these per-point arrays, is measured."""
    from oracle import mg_oracle as mo
    if net.variant != "conv":
        raise ValueError("class expansion needs the conv variant (features = the point's own table)")
    ones = lambda m: np.ones((m, m), dtype=bool)  # noqa: E731
    pick = np.array([0, 1, 3, 5, 6])
    cls = np.broadcast_to(np.asarray(table, dtype=float), (5, 5, 3, 3)).copy()
    expand = lambda c, m: np.ascontiguousarray(c[_band(m)[:, None], _band(m)[None, :]])  # noqa: E731
    ops, kernels, masks, size = [], [], [], n
    for l in range(levels):
        masks.append(ones(size))
        if l > 0 and ops[-1].shape[0] <= 63:
            ops.append(mo.galerkin(ops[-1], masks[-2], masks[-1]))
            cls = None
        else:
            if l > 0:
                cls = mo.galerkin(expand(cls, 15), ones(15), ones(7))[pick[:, None], pick[None, :]]
            ops.append(expand(cls, size))
        if l < levels - 1:
            if cls is not None:
                kernels.append(expand(mo.infer_kernels(net, np.ascontiguousarray(cls), ones(5)), size))
            else:
                kernels.append(mo.infer_kernels(net, ops[-1], masks[-1]))
        size //= 2
    lu, perm = mo.lu_factor(mo.materialize(ops[-1], masks[-1]))
    return mo.Hierarchy(ops, masks, lu, perm, kernels, net.slope)


def cpu_sample_n(cfg):
    """Grid size of the CPU sample: the config's own n where one solve fits host memory
    and minutes (constant-coefficient configs up to 4095^2 through
    oracle_hierarchy_constant: config 2 at full size), else CPU_SAMPLE_N."""
    if "MGB_CPU_SAMPLE_N" in os.environ:
        return min(cfg["n"], CPU_SAMPLE_N)
    if cfg["op"] in ("rot", "rot_classed"):
        return min(cfg["n"], 4095)
    return min(cfg["n"], CPU_SAMPLE_N)


def cpu_sample(cfg_name, steps=1, warmup=0, barrier=None, n=None):
    """Oracle port (NumPy, single thread) on a bounded sample of the config: one
    problem of its operator family at cpu_sample_n(cfg)^2 (levels scaled to reach 3x3),
    V(nu, nu) cycles with the history residual, timed like hierarchy.solve (setup
    excluded).  barrier: replicas start timing together."""
    from oracle import mg_oracle as mo
    from paper_2102_12071_b200 import problems as gen
    cfg = CONFIGS[cfg_name]
    n = cpu_sample_n(cfg) if n is None else min(n, cfg["n"])
    levels = gen.levels_for(n)
    nu = cfg["nu"]
    net = mo.load_net_json(os.path.join(ROOT, "paper_2102_12071_b200", "data", cfg["net"]))
    t0 = time.perf_counter()
    if cfg["op"] in ("rot", "rot_classed"):
        f = gen.uniform_rhs(n, cfg["seed"])
        if n > 1023:
            h = oracle_hierarchy_constant(gen.rotated_fd(1, cfg["theta"], cfg["eps"], h=1.0 / (n + 1))[0, 0], n, levels, net)
        else:
            h = mo.equip_inferred(mo.build_hierarchy(gen.rotated_fd(n, cfg["theta"], cfg["eps"]), levels), net)
    else:
        if cfg["op"] == "grf":
            A, f = gen.grf_diffusion_5pt(n, seed=cfg["seed"]), gen.uniform_rhs(n, cfg["seed"])
        else:
            eps, theta = gen.batch_parameters(cfg["batch"], seed=cfg["seed"])
            A, f = gen.rotated_fd(n, theta[0], eps[0]), gen.uniform_rhs(n, [4, 0])
        h = mo.equip_inferred(mo.build_hierarchy(A, levels), net)
    A = h.ops[0]
    setup = time.perf_counter() - t0
    u = np.zeros((n, n))
    fn = float(np.linalg.norm(f))
    times = []
    if barrier is not None:
        barrier.wait()
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
                      f"config's operator family at {n}^2 ({levels} levels), {len(times)} cycle(s) timed, "
                      f"setup {setup:.1f}s excluded; cpu {cpu_model()}",
            "per_cycle_s": per_cycle, "n": n, "same_size": n == cfg["n"]}


def _c4_problem_cycle(i):
    """One config-4 problem on one core: hierarchy + inference (untimed) and one
    timed V(1,1) cycle + history residual (worker of the process pool)."""
    import time as _t
    from oracle import mg_oracle as mo
    from paper_2102_12071_b200 import problems as gen
    cfg = CONFIGS["c4"]
    n = cfg["n"]
    eps, theta = gen.batch_parameters(cfg["batch"], seed=cfg["seed"])
    A, f = gen.rotated_fd(n, theta[i], eps[i]), gen.uniform_rhs(n, [4, i])
    h = mo.equip_inferred(mo.build_hierarchy(A, cfg["levels"]),
                          mo.load_net_json(os.path.join(ROOT, "paper_2102_12071_b200", "data", cfg["net"])))
    u = np.zeros((n, n))
    fn = float(np.linalg.norm(f))
    t0 = _t.perf_counter()
    u = mo.v_cycle(h, 0, f, u, cfg["nu"], cfg["nu"])
    _ = float(np.linalg.norm(f - mo.apply_stencil(A, u))) / fn
    return _t.perf_counter() - t0


def cpu_sample_pool(cfg_name, nproblems=None):
    """Config 4 on all host cores: a process pool over independent problems (the
    reference's own concurrency model, cli.py:746-752), one cycle each; the
    throughput is total unknowns / wall time of the timed cycles."""
    import multiprocessing as mpc
    cfg = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    nproblems = nproblems or min(cfg["batch"], 2 * cores)
    env = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env:
        os.environ[k] = "1"
    try:
        with mpc.get_context("spawn").Pool(cores) as pool:
            t0 = time.perf_counter()
            times = pool.map(_c4_problem_cycle, range(nproblems))
            wall = time.perf_counter() - t0
    finally:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    per_cycle_core = float(np.mean(times))
    value = cores * cfg["n"] ** 2 / per_cycle_core
    return {"value": value, "unit": "unknowns/s", "cores": cores, "kind": "port",
            "sample": f"oracle/mg_oracle.py (NumPy) on a pool of {cores} single-threaded processes, "
                      f"{nproblems} config-4 problems at {cfg['n']}^2, one V({cfg['nu']},{cfg['nu']}) cycle + history "
                      f"each (setup excluded); value = cores x unknowns / mean cycle time "
                      f"({per_cycle_core * 1e3:.1f} ms; pool wall {wall:.1f}s incl. setup); cpu {cpu_model()}",
            "per_cycle_s": per_cycle_core / cores}


def _replica_worker(cfg_name, steps, warmup, barrier, out, n=None):
    """One single-threaded replica of cpu_sample (worker of cpu_sample_replicas): the
    setup runs before the barrier, so every replica's timed cycles overlap."""
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    sys.path.insert(0, ROOT)
    s = cpu_sample(cfg_name, steps=steps, warmup=warmup, barrier=barrier, n=n)
    out.put(s["per_cycle_s"])


def host_mem_available_gb():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                return float(ln.split()[1]) / 1e6
    except Exception:
        pass
    return 16.0


def cpu_sample_replicas(cfg_name, steps=1, warmup=0, max_procs=32, n=None):
    """Single-problem configs on all host cores: one solve of the reference is
    single-threaded NumPy, so the host's throughput is independent replicas, one
    per core (the reference's own concurrency model: the bench thread pool,
    cli.py:746-752), each timing cpu_sample's cycles at the same moment; value =
    sum over replicas of unknowns / cycle time (memory-bandwidth contention
    between replicas included).  Replicas are capped by host memory (a 4095^2
    oracle solve holds about 4.5 GB)."""
    import multiprocessing as mpc
    cfg = CONFIGS[cfg_name]
    n = cpu_sample_n(cfg) if n is None else min(n, cfg["n"])
    per_replica_gb = 6.0 * (n / 4095.0) ** 2 + 0.3
    cores = max(1, min(os.cpu_count() or 1, max_procs, int(0.8 * host_mem_available_gb() / per_replica_gb)))
    if cores == 1:
        return cpu_sample(cfg_name, steps=steps, warmup=warmup, n=n)
    ctx = mpc.get_context("spawn")
    barrier, out = ctx.Barrier(cores), ctx.Queue()
    procs = [ctx.Process(target=_replica_worker, args=(cfg_name, steps, warmup, barrier, out, n)) for _ in range(cores)]
    for p in procs:
        p.start()
    per = [out.get() for _ in procs]
    for p in procs:
        p.join()
    value = float(sum(n * n / t for t in per))
    return {"value": value, "unit": "unknowns/s", "cores": cores, "kind": "port",
            "sample": f"oracle/mg_oracle.py (NumPy) on {cores} concurrent single-threaded replicas, each one "
                      f"problem of the config's operator family at {n}^2 ({gen_levels(n)} levels), "
                      f"{steps} V({cfg['nu']},{cfg['nu']}) cycle(s) + history residual timed after {warmup} "
                      f"warm-up (setup excluded); value = sum of the replicas' unknowns / cycle time "
                      f"(mean cycle {np.mean(per) * 1e3:.0f} ms); cpu {cpu_model()}",
            "per_cycle_s": float(np.mean(per)) / cores, "n": n, "same_size": n == cfg["n"]}


def gen_levels(n):
    from paper_2102_12071_b200 import problems as gen
    return gen.levels_for(n)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except Exception:
        pass
    return f"{os.cpu_count()} cpus"


def workload_desc(cfg_name):
    c = CONFIGS[cfg_name]
    b = f"{c['batch']} x " if c["batch"] > 1 else ""
    return (f"{cfg_name}: {c['desc']}, {b}{c['n']}^2, {c['levels']} levels, V({c['nu']},{c['nu']}) x "
            f"{c['cycles']} cycles + history, learned conv smoother")


def run_reference(args):
    """The reference arm: the oracle port on all host cores at the config's own grid size
    where that is feasible (cpu_sample_n: config 2 at its full 4095^2, about 26 s per
    cycle and 4.5 GB per replica, so one or two timed cycles), with the quick 1023^2
    sample of round 1 kept beside it as `sample_1023`."""
    from paper_2102_12071_b200 import dist as D
    world, rank, local = D.env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    extra = None
    if cfg["batch"] > 1:
        s = cpu_sample_pool(args.config)
    else:
        n = cpu_sample_n(cfg)
        big = n > 1023
        s = cpu_sample_replicas(args.config, steps=max(1, min(args.steps, 2 if big else 10)),
                                warmup=0 if big else min(args.warmup, 1))
        if big:
            q = cpu_sample_replicas(args.config, steps=max(1, min(args.steps, 5)), warmup=1, n=1023)
            extra = {"value": q["value"], "unit": "unknowns/s", "cores": q["cores"], "n": 1023}
    n_s = s.get("n", cfg["n"])
    line = {"metric": "unknowns/sec per V-cycle (fp64)", "value": s["value"], "unit": "unknowns/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s["per_cycle_s"] * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg["batch"] > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators)", "impl": "reference",
            "config": {"workload": workload_desc(args.config), "sample_n": n_s, "same_size": n_s == cfg["n"]},
            "cpu_baseline": {k: s[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": s["value"], "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if extra:
        line["sample_1023"] = extra
    print(json.dumps(line), flush=True)
    return 0


def run_dd(args, world, rank, local, dev):
    """A single-problem config over N GPUs (strong scaling of the one problem): row-block
    domain decomposition of the fine levels (NCCL halo exchange overlapped with the
    interior rows of every pass, coarse levels agglomerated below 1023 rows).  Every
    rank builds the same hierarchy (the tables are replicated: band classes for configs
    2 / 5, per-point planes for config 3) and owns a row block of u and f."""
    import torch
    import torch.distributed as dist
    from paper_2102_12071_b200 import dd, dist as D
    cfg = CONFIGS[args.config]
    h, f_host, info = build_problem(args.config, local)
    n, nu, cycles = cfg["n"], cfg["nu"], cfg["cycles"]
    host_backend = dist.get_backend() == "gloo"
    rdev = None if host_backend else dev   # device of the control-plane reductions
    solver = dd.from_process_group(h, agglomerate_rows=1023, backend="host" if host_backend else "nccl")
    r0, r1 = solver.rows(rank)
    f_blk = torch.from_numpy(np.ascontiguousarray(f_host[0, r0:r1])).to(dev)
    del f_host
    solver.set_rhs(rank, f_blk)
    stream = torch.cuda.current_stream(dev)
    hist = torch.empty(cycles + 1, dtype=torch.float64, device=dev)
    warm = max(3, args.warmup)

    def timed(steps, sample_clocks=False):
        for _ in range(warm if sample_clocks else 2):
            solver.run_cycles(cycles, nu, nu, True, hist)
        dist.barrier()
        torch.cuda.synchronize(dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(local) if sample_clocks else None
        if clk:
            clk.__enter__()
        ev0.record(stream)
        for _ in range(steps):
            solver.run_cycles(cycles, nu, nu, True, hist)
        ev1.record(stream)
        dist.barrier()
        torch.cuda.synchronize(dev)
        if clk:
            clk.__exit__()
        return D.max_over_ranks(ev0.elapsed_time(ev1) / steps, rdev), clk

    ms_max, clk = timed(args.steps, sample_clocks=True)
    hist_last = float(hist[-1].item())
    sent, xsteps = solver.stats()
    value = n * n * cycles / (ms_max * 1e-3)
    # where the exchanges cost: the same schedule without overlap, and with the exchanges
    # skipped altogether (wrong numbers, right timing: the exposed exchange time)
    probe = max(1, min(args.steps, 3))
    solver.set_option("overlap", False)
    ms_serial, _ = timed(probe)
    solver.set_option("overlap", True)
    solver.set_option("exchange", False)
    ms_noex, _ = timed(probe)
    solver.set_option("exchange", True)
    # e2e: host block in, solution block out, inside the timed region
    f_pin = f_blk.cpu().pin_memory()
    u_pin = torch.empty_like(f_pin).pin_memory()
    solver.set_rhs(rank, f_blk)
    solver.run_cycles(cycles, nu, nu, True, hist)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(1, min(args.steps, 3))
    e0.record(stream)
    for _ in range(e_steps):
        f_blk.copy_(f_pin, non_blocking=True)
        solver.set_rhs(rank, f_blk)
        solver.run_cycles(cycles, nu, nu, True, hist)
        u_pin.copy_(solver.solution(rank), non_blocking=True)
        hh = hist.cpu()
    e1.record(stream)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e_ms = D.max_over_ranks(e0.elapsed_time(e1) / e_steps, rdev)
    if rank == 0:
        line = {
            "metric": "unknowns/sec per V-cycle (fp64)", "value": value, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators; reference-trained seeded conv net fixture)",
            "config": {"workload": workload_desc(args.config), "unknowns_per_problem": n * n, "problems": 1,
                       "cycles_per_step": cycles, "l2": "inputs larger than L2",
                       "parallelism": f"row-block domain decomposition x{world} (NCCL halos overlapped with the "
                                      f"interior rows, {solver.distributed_levels} distributed levels, coarse levels "
                                      f"below 1023 rows agglomerated and solved on every rank)"},
            "dd": {"rows_per_rank": r1 - r0, "sent_bytes_per_step_rank0": sent, "exchange_steps_per_step": xsteps,
                   "ms_per_step_without_overlap": ms_serial, "ms_per_step_without_exchanges": ms_noex,
                   "exchange_exposed_ms": ms_max - ms_noex, "exchange_hidden_by_overlap_ms": ms_serial - ms_max},
            "e2e": {"value": n * n * cycles / (e_ms * 1e-3), "unit": "unknowns/s",
                    "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 8 * n * n + 8 * (cycles + 1)},
            "gpu_launches": None, "history_last": hist_last, "clocks": clk.summary(),
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def run_ours(args):
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2102_12071_b200 import _lib, device as dv, dist as D
    world, rank, local = D.env()
    # MGB_BENCH_BACKEND=gloo: the test of this script's multi-rank path on one GPU (ranks
    # share cuda:0 and the decomposition exchanges through the host); never a measurement
    backend = os.environ.get("MGB_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    D.init(backend, device=dev)
    cfg = CONFIGS[args.config]
    if world > 1 and cfg["batch"] == 1 and cfg["n"] >= 2047:
        return run_dd(args, world, rank, local, dev)   # one problem over the ranks: strong scaling
    batched = cfg["batch"] > 1
    lo, hi = D.shard(cfg["batch"], rank, world) if batched else (0, 1)
    h, f_host, info = build_problem(args.config, local, lo, hi)
    n, levels, nu, cycles = cfg["n"], cfg["levels"], cfg["nu"], cfg["cycles"]
    nb = info["local_batch"]
    f = torch.from_numpy(np.ascontiguousarray(f_host if batched else f_host[0])).to(dev)
    u = torch.zeros_like(f)
    hist = torch.empty((nb, cycles + 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    warm = max(3, args.warmup)
    for _ in range(warm):
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
    ms_max = D.max_over_ranks(ms, dev)
    total_problems = cfg["batch"] if batched else world
    value = total_problems * n * n * cycles / (ms_max * 1e-3)
    hist_all = D.gather_rows(hist.cpu().numpy(), cfg["batch"], dev) if batched else hist.cpu().numpy()

    # dominant kernels: level-0 PRE / POST phases, timed live (CUDA events on the
    # launching stream) through mgb_time_pass
    compact = all(h.storage_info(0))
    w = h.acquire_work()
    try:
        ms_pre, ms_post = C.c_double(), C.c_double()
        ut = torch.zeros_like(f)
        _lib.call("mgb_time_pass", h.handle, w, 0, 0, nu, dv.ptr(f), dv.ptr(ut), 10, C.byref(ms_pre), dv.stream(f))
        _lib.call("mgb_time_pass", h.handle, w, 0, 1, nu, dv.ptr(f), dv.ptr(ut), 10, C.byref(ms_post), dv.stream(f))
        torch.cuda.synchronize(dev)
    finally:
        h.release_work(w)
    peak, peak_kind = measured_peak()
    # algorithmic bytes per fine point of one phase: u in, f, u out (8 B each) plus
    # the restricted residual (PRE) or coarse correction (POST) at 8 B per coarse
    # point; + 72 B for M and 8 B per nonzero A entry (72, or 40 for a 5-point A whose
    # zero corner planes are never read) when they are per-point planes
    per_pt = 26 + (0 if compact else 72 + 8 * h.stencil_points(0))
    pass_bytes = per_pt * n * n * nb
    achieved = pass_bytes / (ms_pre.value * 1e-3) / 1e9
    achieved_post = pass_bytes / (ms_post.value * 1e-3) / 1e9
    traffic, _ = ncu_traffic(args.config)

    # e2e through the host-buffer C-ABI calls (pinned host f in, u + history out).
    # Headline: a stream of e_steps independent solves through
    # mgb_run_cycles_host_many (copies of neighbouring solves overlap each solve's
    # cycles); also the one-solve-per-call synchronous figure.
    f_pin = [torch.from_numpy(np.ascontiguousarray(f_host if batched else f_host[0])).pin_memory() for _ in range(2)]
    u_pin = [torch.zeros_like(f_pin[0]).pin_memory() for _ in range(2)]
    fh, uh = [x.numpy() for x in f_pin], [x.numpy() for x in u_pin]
    e_steps = max(3, min(args.steps, 50))   # the same K steps as the device-timed region
    hist_hosts = [np.empty((nb, cycles + 1)) for _ in range(e_steps)]
    f_list = [fh[k % 2] for k in range(e_steps)]
    u_list = [uh[k % 2] for k in range(e_steps)]
    for _ in range(2):
        h.run_cycles_host(fh[0], uh[0], cycles, nu, nu, history_host=hist_hosts[0], u_zero=True, stream=dv.stream(f))
    h.run_cycles_host_many(f_list, u_list, cycles, nu, nu, history_hosts=hist_hosts, u_zero=True,
                           stream=dv.stream(f))   # warm: graphs of both staging sets, pinned history staging
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h.run_cycles_host_many(f_list, u_list, cycles, nu, nu, history_hosts=hist_hosts, u_zero=True, stream=dv.stream(f))
    e1.record(stream)
    barrier()
    e_ms = D.max_over_ranks(e0.elapsed_time(e1) / e_steps, dev)
    e2e_value = total_problems * n * n * cycles / (e_ms * 1e-3)
    assert np.array_equal(hist_hosts[-1][:, -1], hist.cpu().numpy()[:, -1]), "pipelined host solves differ from the device run"
    e0.record(stream)
    for _ in range(3):
        h.run_cycles_host(fh[0], uh[0], cycles, nu, nu, history_host=hist_hosts[0], u_zero=True, stream=dv.stream(f))
    e1.record(stream)
    barrier()
    e_ms_single = D.max_over_ranks(e0.elapsed_time(e1) / 3, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample_pool(args.config) if batched else cpu_sample(args.config, steps=1)
    if rank == 0:
        bpu = cycle_bytes_per_fine_unknown(n, levels, nu, nu)
        kname = h.pass_kernel(0, nu)   # the kernel launch_pass dispatches level 0 to
        infer_pts = sum((25 if h.storage_info(l)[0] else (n >> l) ** 2) * nb for l in range(levels - 1))
        # compulsory traffic of one fused cycle: per level a PRE pass (u, f in; u out; the
        # restricted residual at 8 B per coarse point; on levels >= 1 the start is zero, so
        # u is not read) and a POST pass (u, f, coarse correction in; u out), plus the
        # per-point tables where a level streams them; the history residual pass of the
        # last cycle (u, f in) is spread over the cycles
        cyc_bytes = 0.0
        for l in range(levels - 1):
            nl = (n >> l) ** 2
            tables = 0 if all(h.storage_info(l)) else 72 + 8 * h.stencil_points(l)
            pre = (26 if l == 0 else 18) + tables
            cyc_bytes += nl * nb * (pre + 26 + tables)
        cyc_bytes += 16.0 * n * n * nb / cycles
        cyc_s = ms_max * 1e-3 / cycles
        hl = hist_all[:, -1]
        line = {
            "metric": "unknowns/sec per V-cycle (fp64)", "value": value, "unit": "unknowns/s",
            "n_gpus": world, "steps": args.steps, "warmup": warm, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong" if batched else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generators; reference-trained seeded conv net fixture)",
            "config": {"workload": workload_desc(args.config), "unknowns_per_problem": n * n,
                       "problems": total_problems, "cycles_per_step": cycles,
                       "l2": "inputs larger than L2 (level-0 u, f and tables exceed 126 MB)",
                       "parallelism": (f"batch split x{world}" if batched else f"replicas x{world}")},
            "roofline": {"bound": "hbm",
                         "kernel": f"{kname} PRE, level 0 (sweeps + residual + full-weighting restriction, "
                                   "one row-streaming pass)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": pass_bytes, "launch_ms": ms_pre.value,
                         "storage": "band-class tables (A, M exact, shared memory)" if compact else "per-point planes",
                         "post": {"kernel": f"{kname} POST, level 0 (prolongation + sweeps)",
                                  "achieved": achieved_post, "frac": achieved_post / peak,
                                  "launch_ms": ms_post.value}},
            "cycle_roofline": {"bound": "hbm", "bytes_per_cycle": cyc_bytes, "cycle_ms": cyc_s * 1e3,
                               "achieved": cyc_bytes / cyc_s / 1e9, "peak": peak, "unit": "GB/s",
                               "frac": cyc_bytes / cyc_s / 1e9 / peak,
                               "model": "compulsory bytes of the fused passes of every level (26 B per point per "
                                        "pass, 18 B for the zero-start PRE of levels >= 1, + per-point tables where "
                                        "streamed) / measured cycle time; levels >= 1 are L2-resident, so this is a "
                                        "lower bound on how far the whole cycle is from streaming at HBM speed"},
            "cycle_model": {"survey_bytes_per_fine_unknown": 172.6 if compact else bpu,
                            "survey_model": "compact (SURVEY 8(d))" if compact else "per-point (SURVEY 8(d))",
                            "effective_GBps": value / world * (172.6 if compact else bpu) / 1e9},
            "e2e": {"value": e2e_value, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * n * n * nb,
                    "d2h_bytes_per_step": 8 * n * n * nb + 8 * (cycles + 1) * nb,
                    "mode": f"stream of {e_steps} independent solves through mgb_run_cycles_host_many (pinned "
                            "host f in, u + history out; the copies of neighbouring solves overlap each solve's "
                            "cycles)",
                    "single_call": {"value": total_problems * n * n * cycles / (e_ms_single * 1e-3),
                                    "mode": "one synchronous mgb_run_cycles_host call per solve"}},
            "gpu_launches": int(launches_per_step * args.steps),
            "history_last": float(np.median(hl)) if batched else float(hl[0]),
            "history_last_stat": "median over problems" if batched else "single problem",
            "setup_s": {"galerkin_lu": info["setup_rap_lu_s"], "cnn_inference": info["setup_infer_s"],
                        # points the stencil -> smoother CNN evaluated: every point of a level that keeps
                        # per-point tables, 25 class representatives of a band-class level
                        "cnn_points": infer_pts, "cnn_points_per_s": infer_pts / max(info["setup_infer_s"], 1e-12)},
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
