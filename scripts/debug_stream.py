import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import device as dv, problems as gen
for n, lv, storage in [(7, 2, "auto"), (7, 2, "planes"), (15, 2, "auto"), (15, 2, "planes"), (31, 3, "auto"), (255, 3, "auto")]:
    A = gen.rotated_fd(n, math.pi / 6, 0.01)
    h = mg.equip_classical(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), lv), "jacobi")
    h.set_storage(storage)
    f = dv.to_dev(gen.uniform_rhs(n, 0))
    out = []
    for fused in (False, True):
        h.set_fused(fused)
        u = dv.zeros(f.shape)
        hist = dv.host(h.run_cycles(f, u, 1, 1, 1, u_zero=True))
        torch.cuda.synchronize()
        out.append((hist, dv.host(u)))
    d = np.abs(out[0][1] - out[1][1])
    print(n, lv, storage, "hist", out[0][0], out[1][0], "maxdiff u", d.max(), flush=True)
    if d.max() > 1e-12:
        np.set_printoptions(linewidth=200, precision=3)
        print(d[:8, :8])
