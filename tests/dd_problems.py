"""Problems of the decomposition tests (shared by test_dd_gpu.py and dd_worker.py):
name -> (device hierarchy, host right-hand side, nu, cycles, agglomerate_rows)."""
import math
import os

import numpy as np

import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import problems as gen

DATA = os.path.join(os.path.dirname(os.path.abspath(mg.__file__)), "data")


def build(name):
    net = mg.load_model(os.path.join(DATA, "net_conv.json"))
    if name == "classed511":      # config-5 family, band-class tables only
        n = 511
        table = gen.rotated_fd(1, math.pi / 3, 0.01, h=1.0 / (n + 1))[0, 0]
        h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net)
        return h, gen.uniform_rhs(n, 11), 2, 3, 127
    if name == "grf1023":         # config-3 family: per-point planes, 5-point level 0
        n = 1023
        A = gen.grf_diffusion_5pt(n, seed=2)
        spec = mg.GridSpec(n, n, 1.0 / n, np.ones((n, n), bool))
        h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(spec, A), gen.levels_for(n)),
                              mg.load_model(os.path.join(DATA, "net_conv_c3.json")))
        return h, gen.uniform_rhs(n, 2), 2, 3, 255
    if name == "lshape511":       # masked domain (per-point planes + masks on every level)
        n = 511
        mask = gen.geometry_mask("lshape", n)
        A = gen.rotated_fd(n, math.pi / 6, 0.01)
        A[~mask] = 0.0
        A[~mask, 1, 1] = 1.0
        spec = mg.GridSpec(n, n, 1.0 / (n + 1), mask)
        h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(spec, A), 6), net)
        return h, gen.uniform_rhs(n, 5) * mask, 1, 3, 127
    if name == "c2_1023":         # config-2 family through build_hierarchy (class-compacted on the device)
        n = 1023
        A = gen.rotated_fd(n, math.pi / 4, 1e-3)
        h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), gen.levels_for(n)),
                              mg.load_model(os.path.join(DATA, "net_conv_c2.json")))
        return h, gen.uniform_rhs(n, 1), 2, 3, 255
    raise KeyError(name)
