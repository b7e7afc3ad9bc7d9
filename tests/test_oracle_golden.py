"""Pin the CPU oracle (oracle/mg_oracle.py) to golden vectors produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from oracle import mg_oracle as mo
from paper_2102_12071_b200 import problems as gen

from cases import LARGE, SMALL, load
from conftest import golden, rel_err

KEYS = ["square9", "lshape9", "cylinder9", "square10"]


@pytest.mark.parametrize("key", KEYS)
def test_apply_stencil_bit_exact(ops_golden, key):
    g = ops_golden
    out = mo.apply_stencil(g[f"{key}_A"], g[f"{key}_u"], g[f"{key}_mask"])
    assert np.array_equal(out, g[f"{key}_Au"])


@pytest.mark.parametrize("key", KEYS)
def test_restrict_prolong_bit_exact(ops_golden, key):
    g = ops_golden
    mask, mc = g[f"{key}_mask"], g[f"{key}_maskc"]
    assert np.array_equal(mo.coarse_mask(mask), mc)
    assert np.array_equal(mo.restrict(g[f"{key}_u"], mc), g[f"{key}_rc"])
    assert np.array_equal(mo.prolong(g[f"{key}_ec"], mask.shape, mask), g[f"{key}_Pe"])


@pytest.mark.parametrize("key", KEYS)
def test_galerkin_bit_exact(ops_golden, key):
    g = ops_golden
    Ac = mo.galerkin(g[f"{key}_A"], g[f"{key}_mask"], g[f"{key}_maskc"])
    assert np.array_equal(Ac, g[f"{key}_Ac"])


@pytest.mark.parametrize("key", KEYS)
def test_lu(ops_golden, key):
    g = ops_golden
    M = mo.materialize(g[f"{key}_Ac"], g[f"{key}_maskc"])
    lu, perm = mo.lu_factor(M)
    assert np.array_equal(perm, g[f"{key}_perm"])
    assert rel_err(lu, g[f"{key}_lu"]) < 1e-14
    assert rel_err(mo.lu_solve(lu, perm, g[f"{key}_lub"]), g[f"{key}_lux"]) < 1e-13


def test_lu_singular_raises():
    M = np.array([[1.0, 2.0], [2.0, 4.0]])
    with pytest.raises(mo.OracleError) as ei:
        mo.lu_factor(M)
    assert ei.value.kind == "SingularMatrixError" and ei.value.pivot_index == 1


def test_problem_generators_match_reference_assembly():
    g = golden("problems.npz")
    for i in range(4):
        n, th, ep = g[f"rot{i}_params"]
        A = gen.rotated_fd(int(n), th, ep)
        assert np.array_equal(A[0, 0], g[f"rot{i}"])


@pytest.mark.parametrize("name", sorted(SMALL))
def test_hierarchy_and_kernels(name, nets):
    c = load(name)
    g = c["golden"]
    h = mo.build_hierarchy(c["A0"], c["levels"], c["mask"])
    for l in range(h.depth):
        assert np.array_equal(h.masks[l], g[f"mask{l}"])
        assert h.ops[l].shape == g[f"A{l}"].shape
        assert rel_err(h.ops[l], g[f"A{l}"]) <= 1e-15
    assert np.array_equal(h.perm, g["coarse_perm"])
    if c["smoother"] == "jacobi":
        mo.equip_jacobi(h)
    else:
        mo.equip_inferred(h, nets[c["smoother"]])
        for l in range(h.depth - 1):
            assert rel_err(h.kernels[l], g[f"K{l}"]) < 1e-13
    u, hist = mo.run_cycles(h, c["f"], c["cycles"], c["nu"], c["nu"])
    gh = g["history"]
    assert np.all(np.abs(hist - gh) <= 1e-12 * np.abs(gh) + 1e-300)
    assert rel_err(u, g["u"]) < 1e-11


def test_v_cycle_nu1_equals_reference_v_cycle(nets):
    """solve() with V(1,1) reproduces the golden V(1,1) history prefix."""
    c = load("case_rot15_jacobi_v11")
    h = mo.equip_jacobi(mo.build_hierarchy(c["A0"], c["levels"], c["mask"]))
    u, hist, it, conv = mo.solve(h, c["f"], tol=1e-30, max_iter=4, raise_on_divergence=False)
    assert it == 4 and not conv
    assert np.allclose(hist, c["golden"]["history"][:5], rtol=1e-12, atol=0)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1_fd_conv", "c1_q1_conv"])
def test_config1_history(name, nets):
    c = load(name)
    g = c["golden"]
    h = mo.equip_inferred(mo.build_hierarchy(c["A0"], c["levels"]), nets["conv"])
    for l in range(h.depth):
        assert rel_err(g[f"Asum{l}"], [h.ops[l].sum(), np.abs(h.ops[l]).sum()]) < 1e-12
    for l in range(h.depth - 1):
        K = h.kernels[l]
        assert rel_err(K[K.shape[0] // 2, K.shape[1] // 2], g[f"Kmid{l}"]) < 1e-13
        assert rel_err(K[0, 0], g[f"Kcorner{l}"]) < 1e-13
    u, hist = mo.run_cycles(h, c["f"], c["cycles"], c["nu"], c["nu"])
    assert np.all(np.abs(hist - g["history"]) <= 1e-10 * np.abs(g["history"]))
    assert rel_err(u, g["u"]) < 1e-10


# ---------------------------------------------------------------------------
# Krylov (krylov.py): the oracle's fgmres / gmres against the reference's runs

from krylov_cases import krylov_case, krylov_names  # noqa: E402


@pytest.mark.parametrize("name", krylov_names())
def test_krylov_oracle_matches_reference(name, nets):
    c = krylov_case(name)
    mask = c["mask"]
    act = mo.grid_action(c["A"], mask)
    pc = None
    if c["nu"] > 0:
        h = mo.build_hierarchy(c["A"], 4, mask)
        h = mo.equip_jacobi(h) if c["smoother"] == "jacobi" else mo.equip_inferred(h, nets["conv"])
        pc = mo.cycle_preconditioner(h, c["nu"], c["nu"])
    if c["method"] == "fgmres":
        u, it, hist, conv = mo.fgmres(act, c["f"], pc, c["tol"], c["max_iter"], c["restart"])
    else:
        u, it, hist, conv = mo.gmres(act, c["f"], c["tol"], c["max_iter"], c["restart"])
    assert it == c["iterations"] and conv == c["converged"]
    assert len(hist) == len(c["history"])
    assert np.allclose(hist, c["history"], rtol=1e-12, atol=0), np.max(np.abs(np.array(hist) / c["history"] - 1))
    assert rel_err(u, c["u"]) <= 1e-11


def test_fgmres_config_validation():
    import paper_2102_12071_b200 as mg
    with pytest.raises(mg.ConfigError):
        mg.FgmresConfig(tol=0.0)
    with pytest.raises(mg.ConfigError):
        mg.FgmresConfig(restart=0)
    with pytest.raises(mg.ConfigError):
        mg.FgmresConfig(max_iter=0)


# ---------------------------------------------------------------------------
# shared-kernel conv smoother (smoothers.py:105-178): oracle vs reference

import conv_cases as cc  # noqa: E402


def _osm(prefix):
    form, layers, skip, act, slope, gain = cc.params(prefix)
    return mo.ConvSm(list(layers), skip, act, slope, gain)


@pytest.mark.parametrize("g", ["square", "lshape"])
def test_convolve_and_conv_apply_bit_exact(g):
    z = cc.conv_golden()
    mask = z[f"convolve/{g}/mask"]
    assert np.array_equal(mo.convolve(z[f"convolve/{g}/w"], z[f"convolve/{g}/u"], mask), z[f"convolve/{g}/out"])
    for key in [k for k in cc.names("apply") if k.startswith(g)]:
        pre = f"apply/{key}"
        assert np.array_equal(mo.conv_apply(_osm(pre), z[f"{pre}/r"], mask), z[f"{pre}/out"]), key
        if f"{pre}/effective" in z.files:
            assert np.allclose(mo.effective_kernel(_osm(pre)), z[f"{pre}/effective"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", cc.names("cycle"))
def test_conv_smoother_cycles_oracle(name):
    z = cc.conv_golden()
    pre = f"cycle/{name}"
    A, mask, f, nu = z[f"{pre}/A0"], z[f"{pre}/mask"], z[f"{pre}/f"], int(z[f"{pre}/nu"])
    h = mo.build_hierarchy(A, 4, mask)
    h.kernels = [_osm(f"{pre}/L{l}") for l in range(3)]
    if name.startswith("init"):
        for l in range(3):   # equip_conv_init restated
            ref, mine = h.kernels[l], mo.conv_init(h.ops[l], h.masks[l])
            assert ref.gain == mine.gain and all(np.array_equal(a, b) for a, b in zip(ref.layers, mine.layers))
    u, hist = mo.run_cycles(h, f, 8, nu, nu)
    assert np.allclose(hist, z[f"{pre}/history"], rtol=1e-13, atol=0)
    assert rel_err(u, z[f"{pre}/u"]) <= 1e-12


def test_conv_smoother_model_json_round_trip(tmp_path):
    import paper_2102_12071_b200 as mg
    form, layers, skip, act, slope, gain = cc.params("apply/square/full_leaky")
    spec = mg.full_spec(23)
    sm = mg.ConvSmoother(spec, form, [mg.ConvKernel(w) for w in layers], mg.ConvKernel(skip), act, slope, gain)
    mg.save_model(tmp_path / "c.json", sm, {"note": "round trip"})
    back = mg.load_model(tmp_path / "c.json")
    assert back.form == "full" and back.activation == "leaky" and back.gain == gain
    assert all(np.array_equal(a.weights, b.weights) for a, b in zip(back.layers, sm.layers))
    with pytest.raises(mg.ConfigError):
        mg.ConvSmoother(spec, "full", sm.layers[:2], None)
