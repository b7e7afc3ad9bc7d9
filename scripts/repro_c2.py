"""Reproducibility probe: two identical 3-cycle c2 solves must agree bitwise."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import device as dv, problems as gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4095
lv = gen.levels_for(n)
A = gen.rotated_fd(n, math.pi / 4, 1e-3)
net = mg.load_model(os.path.join(os.path.dirname(mg.__file__), "data", "net_conv_c2.json"))
h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), lv), net)
f = dv.to_dev(gen.uniform_rhs(n, 1))
us = []
for k in range(3):
    u = dv.zeros(f.shape)
    h.run_cycles(f, u, 3, 2, 2, u_zero=True)
    us.append(u)
for k in (1, 2):
    d = (us[k] != us[0])
    print("run", k, "differs at", int(d.sum()), "points; rows", torch.nonzero(d.any(1)).flatten()[:12].tolist(),
          "cols", torch.nonzero(d.any(0)).flatten()[:12].tolist(), "max", float((us[k] - us[0]).abs().max()))
