"""Registry of the golden hierarchy cases written by tests/golden/make_golden.py.

Small cases store A0 / f / per-level A, K in their .npz; large cases
(config 1 at 255^2, config 4 samples at 511^2) store only history, u and
checksums, and rebuild A0 / f from the seeded generators below."""

import math
import os

import numpy as np

from paper_2102_12071_b200 import problems as gen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# name -> (smoother, nu, cycles, levels)
SMALL = {
    "case_rot15_conv_v22": ("conv", 2, 10, 3),
    "case_rot15_jacobi_v11": ("jacobi", 1, 10, 3),
    "case_rot15_convk2_v11": ("conv_k2", 1, 6, 3),
    "case_rot31_fc_v22": ("fc", 2, 8, 4),
    "case_lshape31_conv_v11": ("conv", 1, 8, 4),
    "case_cyl31_fc_v11": ("fc", 1, 6, 3),
    "case_var31_conv_v22": ("conv", 2, 8, 4),
    "case_grf63_conv_v22": ("conv", 2, 8, 5),
    "case_rect20x27_conv_v11": ("conv", 1, 6, 3),
}


def _c4(i):
    eps, theta = gen.batch_parameters(256, seed=3)
    n = 511
    return gen.rotated_fd(n, theta[i], eps[i]), gen.uniform_rhs(n, [4, i])


LARGE = {
    "c1_fd_conv": (lambda: (gen.rotated_fd(255, math.pi / 6, 0.01), gen.uniform_rhs(255, 0)), "conv", 2, 20, 7),
    "c1_q1_conv": (lambda: (gen.rotated_q1(255, math.pi / 6, 0.01), gen.uniform_rhs(255, 0)), "conv", 2, 20, 7),
    "c4_p0": (lambda: _c4(0), "conv", 1, 10, 8),
    "c4_p1": (lambda: _c4(1), "conv", 1, 10, 8),
}


def load(name):
    """Return dict(A0, mask, f, smoother, nu, cycles, levels, golden)."""
    g = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    if name in SMALL:
        sm, nu, cyc, lv = SMALL[name]
        A0, mask, f = g["A0"], g["mask"], g["f"]
    else:
        make, sm, nu, cyc, lv = LARGE[name]
        A0, f = make()
        mask = np.ones(f.shape, dtype=bool)
    return dict(A0=A0, mask=mask, f=f, smoother=sm, nu=nu, cycles=cyc, levels=lv, golden=g)
