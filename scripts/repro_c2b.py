"""Dump u after 1 cycle (zero start) to /tmp/u_<tag>.pt, or compare two dumps."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if sys.argv[1] == "cmp":
    a, b = torch.load(f"/tmp/u_{sys.argv[2]}.pt"), torch.load(f"/tmp/u_{sys.argv[3]}.pt")
    d = a != b
    rows = torch.nonzero(d.any(1)).flatten()
    cols = torch.nonzero(d.any(0)).flatten()
    print("differs at", int(d.sum()), "rows", len(rows), rows[:40].tolist(), "cols", len(cols), cols[:20].tolist(),
          "max", float((a - b).abs().max()))
    sys.exit(0)
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import device as dv, problems as gen
n, cyc = 4095, int(sys.argv[2])
A = gen.rotated_fd(n, math.pi / 4, 1e-3)
net = mg.load_model(os.path.join(os.path.dirname(mg.__file__), "data", "net_conv_c2.json"))
h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), 11), net)
f = dv.to_dev(gen.uniform_rhs(n, 1))
u = dv.zeros(f.shape)
h.run_cycles(f, u, cyc, 2, 2, u_zero=True)
torch.save(u.cpu(), f"/tmp/u_{sys.argv[1]}.pt")
u2 = dv.zeros(f.shape)
h.run_cycles(f, u2, cyc, 2, 2, u_zero=True)
torch.save(u2.cpu(), f"/tmp/u_{sys.argv[1]}b.pt")
