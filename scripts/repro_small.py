import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import device as dv, problems as gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 63
A = gen.rotated_fd(n, math.pi / 6, 0.01)
h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), gen.levels_for(n)),
                      mg.load_model("paper_2102_12071_b200/data/net_conv.json"))
f = dv.to_dev(gen.uniform_rhs(n, 0)); u = dv.zeros(f.shape)
print(dv.host(h.run_cycles(f, u, 2, 2, 2, u_zero=True)))
