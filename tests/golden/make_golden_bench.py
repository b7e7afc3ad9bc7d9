"""Golden vectors at the BENCHMARKED configurations, produced by the UNMODIFIED
reference (mgsmooth 0.1.0).  Build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bench.py [name ...]

The inputs are bench.py's own generators (bench.CONFIGS / bench.operators), so the
GPU tests compare the benchmarked workloads themselves with the reference:

    bench_c2_full.npz   config 2 at its full size: 4095^2 rotated FD (eps=1e-3,
                        theta=pi/4), 11 levels, net_conv_c2, b = U[-1,1] seed 1,
                        3 V(2,2) cycles.  Stores the history, u checksums (sum,
                        sum |u|, sum u^2), the strided subsample u[::64, ::64], the
                        rows 0, n//2, n-1 and columns 0, n-1, per-level operator and
                        kernel checksums.
    bench_c3_511.npz    config 3's family (exp(GRF) 5-point cell-centred, corr.
    bench_c3_1023.npz   length 1/32, seed 2, h = 1/n) at 511^2 / 1023^2 with
                        net_conv_c3, V(2,2), 6 / 4 cycles; full u at 511^2.
    bench_c5_2047.npz   config 5's family (rotated FD eps=0.01, theta=pi/3, seed 5)
                        at 2047^2 (10 levels), net_conv_c5, V(2,2), 4 cycles.

Every hierarchy is the reference's build_hierarchy + equip_inferred with the
V(nu, nu) smoother RepeatedSmoother (cli.py:365-377) and the fixed-count cycle
loop of hierarchy.solve (hierarchy.py:119-146).
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from mgsmooth import grid as rg, hierarchy as rh, smoothers as rs   # noqa: E402  (reference)
from mgsmooth.cli import RepeatedSmoother                              # noqa: E402

import bench                                                           # noqa: E402  (generators only)
from paper_2102_12071_b200 import problems as gen                      # noqa: E402


def checksums(u):
    return np.array([u.sum(), np.abs(u).sum(), (u * u).sum()])


def run(name, A, f, h, levels, net, nu, cycles, full_u=False):
    t0 = time.time()
    n = f.shape[0]
    spec = rg.GridSpec(n, f.shape[1], h, np.ones(f.shape, bool))
    S = rg.StencilField(spec, A)
    hier = rh.build_hierarchy(S, levels)
    t1 = time.time()
    rh.equip_inferred(hier, net)
    t2 = time.time()
    d = {"levels": levels, "nu": nu, "cycles": cycles, "h": h, "n": n}
    for l, lev in enumerate(hier.levels):
        Ad = lev.operator.data
        d[f"Asum{l}"] = np.array([Ad.sum(), np.abs(Ad).sum()])
        d[f"Amid{l}"] = Ad[Ad.shape[0] // 2, Ad.shape[1] // 2]
        d[f"Acorner{l}"] = Ad[0, 0]
        sm = lev.smoother
        if sm is not None:
            K = sm.kernels
            d[f"Ksum{l}"] = np.array([K.sum(), np.abs(K).sum()])
            d[f"Kmid{l}"] = K[K.shape[0] // 2, K.shape[1] // 2]
            d[f"Kcorner{l}"] = K[0, 0]
            lev.smoother = RepeatedSmoother(sm, lev.operator, nu) if nu > 1 else sm
    F = rg.GridFunction(spec, f)
    u = rg.zeros(spec)
    denom = F.norm() if F.norm() > 0 else 1.0
    hist = [(F - rg.apply_stencil(S, u)).norm() / denom]
    for c in range(cycles):
        u = rh.v_cycle(hier, 0, F, u)
        hist.append((F - rg.apply_stencil(S, u)).norm() / denom)
        print(f"  {name} cycle {c + 1}: {hist[-1]:.6e} ({time.time() - t2:.0f}s)", flush=True)
    U = u.values
    d["history"] = np.array(hist)
    d["u_checksums"] = checksums(U)
    d["u_stride64"] = U[::64, ::64].copy()
    d["u_rows"] = U[[0, n // 2, n - 1]].copy()
    d["u_cols"] = U[:, [0, U.shape[1] - 1]].T.copy()
    if full_u:
        d["u"] = U
    d["times_s"] = np.array([t1 - t0, t2 - t1, time.time() - t2])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"{name}: hist[-1]={hist[-1]:.6e}  rap {t1 - t0:.0f}s  infer {t2 - t1:.0f}s  "
          f"cycles {time.time() - t2:.0f}s", flush=True)


def net(fname):
    return rs.load_model(os.path.join(HERE, fname))


def c2_full():
    cfg = bench.CONFIGS["c2"]
    n = cfg["n"]
    A = gen.rotated_fd(n, cfg["theta"], cfg["eps"])
    f = gen.uniform_rhs(n, cfg["seed"])
    run("bench_c2_full", A, f, 1.0 / (n + 1), cfg["levels"], net(cfg["net"]), cfg["nu"], 3)


def c3(n, cycles, full_u):
    cfg = bench.CONFIGS["c3"]
    A = gen.grf_diffusion_5pt(n, seed=cfg["seed"])
    f = gen.uniform_rhs(n, cfg["seed"])
    run(f"bench_c3_{n}", A, f, 1.0 / n, gen.levels_for(n), net(cfg["net"]), cfg["nu"], cycles, full_u)


def c5(n, cycles):
    cfg = bench.CONFIGS["c5"]
    A = gen.rotated_fd(n, cfg["theta"], cfg["eps"])
    f = gen.uniform_rhs(n, cfg["seed"])
    run(f"bench_c5_{n}", A, f, 1.0 / (n + 1), gen.levels_for(n), net(cfg["net"]), cfg["nu"], cycles)


JOBS = {
    "c3_511": lambda: c3(511, 6, True),
    "c3_1023": lambda: c3(1023, 4, False),
    "c5_2047": lambda: c5(2047, 4),
    "c2_full": c2_full,
}


def main():
    names = sys.argv[1:] or list(JOBS)
    for nm in names:
        JOBS[nm]()


if __name__ == "__main__":
    main()
