"""Per-iteration time of hierarchy.solve's device loop (mgb_solve: one graph launch and one
host read of the residual per iteration) on a bench config, against the run_cycles rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2102_12071_b200 as mg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
h, f_host, info = bench.build_problem(cfg, 0)
nu = info["nu"]
for lev in h.levels[:-1]:
    lev.smoother = mg.RepeatedSmoother(lev.smoother, None, nu)
f = torch.from_numpy(np.ascontiguousarray(f_host[0])).cuda()
for _ in range(2):
    u = torch.zeros_like(f)
    rep = h.solve_device(f, u, tol=1e-6, max_iter=40)
n = f.shape[0]
print(f"{cfg}: {rep.iterations} iterations, converged {rep.converged}, residual {rep.residual_history[-1]:.3e}, "
      f"{rep.wall_time / rep.iterations * 1e6:.1f} us per iteration, "
      f"{n * n * rep.iterations / rep.wall_time:.3e} unknowns/s per V-cycle")
