"""Shared-kernel convolutional smoother on the GPU (csrc/mgb_conv.cu) against the
reference (tests/golden/conv.npz): convolve and ConvSmoother.apply bit-exact,
V-cycles with conv smoothers within 1e-10 (SURVEY §8(c) gate (i))."""

import math

import numpy as np
import pytest

import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import problems as gen

import conv_cases as cc
from conftest import rel_err

pytestmark = pytest.mark.gpu


def _sm(spec, prefix):
    form, layers, skip, act, slope, gain = cc.params(prefix)
    return mg.ConvSmoother(spec, form, [mg.ConvKernel(w) for w in layers],
                           None if skip is None else mg.ConvKernel(skip), act, slope, gain)


def _spec(mask):
    n = mask.shape[0]
    return mg.GridSpec(n, mask.shape[1], 1.0 / (n + 1), mask)


@pytest.mark.parametrize("g", ["square", "lshape"])
def test_convolve_and_apply_bit_exact(g):
    z = cc.conv_golden()
    mask = z[f"convolve/{g}/mask"]
    spec = _spec(mask)
    u = mg.GridFunction(spec, z[f"convolve/{g}/u"])
    assert np.array_equal(mg.convolve(mg.ConvKernel(z[f"convolve/{g}/w"]), u).values, z[f"convolve/{g}/out"])
    for key in [k for k in cc.names("apply") if k.startswith(g)]:
        pre = f"apply/{key}"
        sm = _sm(spec, pre)
        out = sm.apply(mg.GridFunction(spec, z[f"{pre}/r"])).values
        assert np.array_equal(out, z[f"{pre}/out"]), key
        if f"{pre}/effective" in z.files:
            assert np.array_equal(mg.effective_kernel(sm).weights, z[f"{pre}/effective"])


@pytest.mark.parametrize("name", cc.names("cycle"))
def test_conv_smoother_cycles_match_reference(name):
    from paper_2102_12071_b200 import device as dv
    z = cc.conv_golden()
    pre = f"cycle/{name}"
    mask, nu = z[f"{pre}/mask"], int(z[f"{pre}/nu"])
    spec = _spec(mask)
    h = mg.build_hierarchy(mg.StencilField(spec, z[f"{pre}/A0"]), 4)
    if name.startswith("init"):
        mg.equip_conv_init(h)
        for l in range(3):
            assert h.levels[l].smoother.gain == float(z[f"{pre}/L{l}/gain"])
    else:
        for l in range(3):
            h.levels[l].smoother = _sm(h.levels[l].spec, f"{pre}/L{l}")
    f = dv.to_dev(z[f"{pre}/f"])
    u = dv.zeros(f.shape)
    hist = dv.host(h.run_cycles(f, u, 8, nu, nu, u_zero=True))[0]
    g = z[f"{pre}/history"]
    assert np.all(np.abs(hist - g) <= 1e-10 * g + 1e-14), np.max(np.abs(hist / g - 1))
    assert rel_err(dv.host(u), z[f"{pre}/u"]) <= 1e-10


def test_equip_trained_transport():
    from paper_2102_12071_b200 import device as dv
    z = cc.conv_golden()
    src = mg.build_hierarchy(mg.StencilField(mg.full_spec(15), gen.rotated_fd(15, math.pi / 6, 0.01)), 3)
    for l in range(2):
        src.levels[l].smoother = _sm(src.levels[l].spec, f"transport/src/L{l}")
    n = 31
    A = gen.rotated_fd(n, math.pi / 6, 0.01)
    tgt = mg.equip_trained(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), 4), src)
    for l in range(3):
        assert tgt.levels[l].smoother.gain == pytest.approx(float(z[f"transport/tgt/L{l}/gain"]), rel=1e-15)
    f = dv.to_dev(gen.uniform_rhs(n, 12))
    u = dv.zeros(f.shape)
    hist = dv.host(tgt.run_cycles(f, u, 6, 1, 1, u_zero=True))[0]
    g = z["transport/history"]
    assert np.all(np.abs(hist - g) <= 1e-10 * g + 1e-14)
    assert rel_err(dv.host(u), z["transport/u"]) <= 1e-10


def test_conv_and_inferred_levels_mix():
    """Per-level smoother kinds can differ: conv smoothers on some levels, per-point
    kernels on others (the cycle dispatches per level)."""
    from paper_2102_12071_b200 import device as dv
    z = cc.conv_golden()
    pre = "cycle/full_lin_v22"
    spec = _spec(z[f"{pre}/mask"])
    h = mg.build_hierarchy(mg.StencilField(spec, z[f"{pre}/A0"]), 4)
    mg.equip_classical(h, "jacobi")
    h.levels[1].smoother = _sm(h.levels[1].spec, f"{pre}/L1")
    f = dv.to_dev(z[f"{pre}/f"])
    u = dv.zeros(f.shape)
    hist = dv.host(h.run_cycles(f, u, 6, 1, 1, u_zero=True))[0]
    assert np.all(np.diff(hist) < 0)
    # swap back to per-point kernels on level 1: the conv smoother is replaced
    mg.equip_classical(h, "jacobi")
    u2 = dv.zeros(f.shape)
    h2 = dv.host(h.run_cycles(f, u2, 6, 1, 1, u_zero=True))[0]
    assert not np.array_equal(hist, h2)
