"""Per-case deviation of device FGMRES/GMRES histories from the reference fixtures."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_2102_12071_b200 as mg
from krylov_cases import krylov_case, krylov_names
from test_krylov_gpu import _setup
for name in krylov_names():
    c = krylov_case(name)
    S, pc = _setup(c)
    cfg = mg.FgmresConfig(tol=c["tol"], max_iter=c["max_iter"], restart=c["restart"])
    if c["method"] == "fgmres":
        u, rep = mg.fgmres(mg.grid_action(S), c["f"], precond=pc, cfg=cfg)
    else:
        u, rep = mg.gmres(mg.grid_action(S), c["f"], cfg=cfg)
    h, g = np.asarray(rep.history), c["history"]
    d = np.abs(h - g)
    print(f"{name:18s} it {rep.iterations}/{c['iterations']} rel max {np.max(d / g):.2e} at {np.argmax(d / g)} "
          f"(g={g[np.argmax(d/g)]:.2e}, g0={g[0]:.2e}) abs/g0 max {np.max(d) / g[0]:.2e} "
          f"u rel {np.linalg.norm(u - c['u']) / np.linalg.norm(c['u']):.2e}")
